mkdir -p gpurun_out
for v in "LRS_SKIP=4" "LRS_SKIP=1" "LRS_NO_CORE=1" "X=1"; do
env $v LRS_NO_AUTOTUNE=1 timeout 120 python tools/cp_debug.py > gpurun_out/cpdbg_$v.log 2>&1; echo "$v rc=$? $(tail -1 gpurun_out/cpdbg_$v.log)"
done
timeout 120 python tools/gpu_debug.py c2_bf16 > gpurun_out/dbg73_c2.log 2>&1; echo "tucker rc=$?"; tail -3 gpurun_out/dbg73_c2.log
