for d in 0 4; do
LRS_CORE_DBG=$d timeout 300 python tools/core_sweep.py c2_bf16 2,7,36 1,7 > gpurun_out/cs88_$d.log 2>&1; echo "dbg=$d"; cat gpurun_out/cs88_$d.log
done
