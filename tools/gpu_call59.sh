mkdir -p gpurun_out
timeout 1200 python tools/core_sweep.py c2_bf16 2,7,36,2 1,7,0,1 2,7,0,1 1,7,84,4 2,7,84,4 1,14,84,4 1,7,68,3 2,7,68,3 1,7,116,7 2,7,116,7 1,7,100,7 1,7,0,7 1,4,116,7 > gpurun_out/plan_sweep59_c2.log 2>&1; echo "rc=$?"
cat gpurun_out/plan_sweep59_c2.log
