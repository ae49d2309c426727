mkdir -p gpurun_out
timeout 120 python tools/gpu_debug.py c3 16 > gpurun_out/dbg6.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wconv -c 1 -o gpurun_out/prof_wconv_c3_16 python tools/gpu_debug.py c3 16 > gpurun_out/ncu6.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu6.log
