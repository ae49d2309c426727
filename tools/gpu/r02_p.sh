mkdir -p gpurun_out/r02p; O=gpurun_out/r02p
LRS_WCONV_DEBUG=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1
timeout 120 python tools/wtrace.py c3 > $O/wtrace_c3.log 2>&1
LRS_EXPERIMENTS=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build2.log 2>&1
timeout 300 python tools/ablate.py c3 "LRS_SKIP=1" "LRS_SKIP=1 LRS_WCONV_DBG=1" "LRS_SKIP=1 LRS_WCONV_DBG=66" "LRS_SKIP=1 LRS_WCONV_DBG=67" "LRS_SKIP=1 LRS_WCONV_DBG=8" > $O/ablate_c3.log 2>&1
grep -v "^\[lrs\]" $O/ablate_c3.log
