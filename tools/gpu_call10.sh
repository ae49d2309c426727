mkdir -p gpurun_out; rm -f gpurun_out/dbg10.log
for d in 0 1 2 4 3 6 5 7; do echo "dbg=$d" >> gpurun_out/dbg10.log; LRS_SPADD_DBG=$d timeout 120 python tools/gpu_debug.py c2_f32 2>&1 | grep forward >> gpurun_out/dbg10.log; done
cat gpurun_out/dbg10.log
