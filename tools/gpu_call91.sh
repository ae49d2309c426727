LRS_WCONV_DEBUG=1 python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
for d in 0 1024 16; do
LRS_WCONV_DBG=$d timeout 300 python tools/core_sweep.py c2_bf16 2,7,36 > gpurun_out/e91_$d.log 2>&1; echo "dbg=$d $(tail -1 gpurun_out/e91_$d.log)"
LRS_WCONV_DBG=$d timeout 300 python tools/core_sweep.py c4 1,1 > gpurun_out/e91c4_$d.log 2>&1; echo "c4 dbg=$d $(head -1 gpurun_out/e91c4_$d.log)"
done
python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
