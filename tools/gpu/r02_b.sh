# round 2, call B: timing ablations (experiment build) of C3 / C4 / C2 + wconv trace of C3
mkdir -p gpurun_out/r02b; O=gpurun_out/r02b
LRS_EXPERIMENTS=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1 || exit 1
for c in c3 c4 c2_bf16; do
timeout 300 python tools/ablate.py $c base "LRS_SKIP=1" "LRS_SKIP=4" "LRS_SKIP=1 LRS_WCONV_DBG=1" "LRS_SKIP=1 LRS_WCONV_DBG=8" \
  "LRS_SKIP=1 LRS_WCONV_DBG=2" "LRS_SKIP=1 LRS_WCONV_DBG=64" "LRS_SKIP=1 LRS_WCONV_DBG=66" "LRS_SKIP=1 LRS_WCONV_DBG=16" \
  "LRS_SKIP=1 LRS_WCONV_DBG=67" "LRS_NO_PDL=1" > $O/ablate_$c.log 2>&1
done
LRS_WCONV_DBG=0 timeout 120 python tools/wtrace.py c3 > $O/wtrace_c3.log 2>&1
timeout 120 python tools/wtrace.py c4 > $O/wtrace_c4.log 2>&1
tail -n 3 $O/*.log
