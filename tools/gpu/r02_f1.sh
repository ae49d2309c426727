mkdir -p gpurun_out/r02f1; O=gpurun_out/r02f1
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_f32 base "LRS_F32_FUSED=1" "CFG_density=0.0" "LRS_F32_FUSED=1 CFG_density=0.0" > $O/ablate.log 2>&1
grep "c2_f32 \[" $O/ablate.log
