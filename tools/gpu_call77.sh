mkdir -p gpurun_out
LRS_VERBOSE=1 timeout 300 python bench.py --config c3 --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/b77.json 2> gpurun_out/b77.err; grep "wconv plan\|core:" gpurun_out/b77.err | tail -2
LRS_WCONV_DEBUG=1 python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
timeout 120 python tools/wtrace.py c3 > gpurun_out/wtrace77_c3.log 2>&1; head -12 gpurun_out/wtrace77_c3.log | cut -c1-600
for dbg in 0 16 1; do
LRS_WCONV_DBG=$dbg timeout 300 python tools/core_sweep.py c3 3,7 > gpurun_out/c3dbg_$dbg.log 2>&1; echo "dbg=$dbg $(tail -1 gpurun_out/c3dbg_$dbg.log)"
done
python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
