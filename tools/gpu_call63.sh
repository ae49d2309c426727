mkdir -p gpurun_out
LRS_WCONV_DEBUG=1 python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
for dbg in 0 16; do
LRS_WCONV_DBG=$dbg timeout 300 python tools/core_sweep.py c2_bf16 2,7,36 > gpurun_out/dbg63_$dbg.log 2>&1; echo "dbg=$dbg"; cat gpurun_out/dbg63_$dbg.log
done
python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
