mkdir -p gpurun_out
timeout 120 python tools/gpu_debug.py c4 > gpurun_out/ncu_plain_c4.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wconv -s 2 -c 1 -o gpurun_out/prof_wconv_c4 python tools/gpu_debug.py c4 > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 120 python tools/gpu_debug.py c3 > gpurun_out/ncu_plain_c3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wconv -s 2 -c 1 -o gpurun_out/prof_wconv_c3 python tools/gpu_debug.py c3 > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
