mkdir -p gpurun_out/r02g4; O=gpurun_out/r02g4
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_CORE_GRID=20" "LRS_CORE_GRID=40" "LRS_CORE_GRID=74" "LRS_CORE_GRID=148" > $O/ablate_c3.log 2>&1
grep "autotune\|core plan\|c3 \[" $O/ablate_c3.log | head -40
