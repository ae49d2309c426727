mkdir -p gpurun_out
./tools/ubench_sparse > gpurun_out/ubench.log 2>&1; echo "ubench rc=$?" >> gpurun_out/rc1.txt
timeout 300 python tools/gpu_debug.py c2_bf16 > gpurun_out/dbg_c2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lrs_gemm -c 3 -o gpurun_out/prof_c2_old python tools/gpu_debug.py c2_bf16 > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/rc1.txt
cat gpurun_out/rc1.txt
