mkdir -p gpurun_out/r02i; O=gpurun_out/r02i
LRS_EXPERIMENTS=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1 || exit 1
timeout 300 python tools/ablate.py c4 base "LRS_SKIP=1" "LRS_SKIP=1 LRS_PW_DBG=1" "LRS_SKIP=1 LRS_PW_DBG=2" "LRS_SKIP=1 LRS_PW_DBG=4" "LRS_SKIP=1 LRS_PW_DBG=3" "LRS_SKIP=1 LRS_PW_DBG=6" "LRS_SKIP=1 LRS_PW_DBG=7" "LRS_SKIP=4" > $O/ablate_c4.log 2>&1
grep -v "^\[lrs\]" $O/ablate_c4.log
