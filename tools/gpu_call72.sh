mkdir -p gpurun_out
LRS_NO_AUTOTUNE=1 LRS_VERBOSE=1 timeout 120 python tools/cp_debug.py > gpurun_out/cpdbg.log 2>&1; echo "rc=$?"
tail -12 gpurun_out/cpdbg.log
