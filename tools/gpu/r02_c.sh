# round 2, call C: timing ablations (experiment build) of C3 / C4 / C2 + core trace of C3
mkdir -p gpurun_out/r02c; O=gpurun_out/r02c
LRS_EXPERIMENTS=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1 || exit 1
for c in c3 c4 c2_bf16; do
timeout 300 python tools/ablate.py $c base "LRS_SKIP=1" "LRS_SKIP=4" "LRS_SKIP=1 LRS_WCONV_DBG=1" "LRS_SKIP=1 LRS_WCONV_DBG=8" \
  "LRS_SKIP=1 LRS_WCONV_DBG=2" "LRS_SKIP=1 LRS_WCONV_DBG=64" "LRS_SKIP=1 LRS_WCONV_DBG=66" "LRS_SKIP=1 LRS_WCONV_DBG=16" \
  "LRS_SKIP=1 LRS_WCONV_DBG=67" "LRS_NO_PDL=1" "LRS_CORE_DBG=4 LRS_SKIP=4" > $O/ablate_$c.log 2>&1
done
timeout 120 python tools/ctrace.py c3 > $O/ctrace_c3.log 2>&1
LRS_VERBOSE=1 timeout 120 python tools/ablate.py c3 base > $O/verbose_c3.log 2>&1
tail -n 15 $O/*.log
