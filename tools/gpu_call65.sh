mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_core_fused.py tests/test_gpu_parity.py -q > gpurun_out/t65.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/t65.log
for c in c2_bf16 c3; do
LRS_VERBOSE=1 timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b65_$c.json 2> gpurun_out/b65_$c.err; echo "$c rc=$?"; tail -1 gpurun_out/b65_$c.json | cut -c140-200; grep autotune gpurun_out/b65_$c.err
done
timeout 600 python tools/core_sweep.py c2_bf16 2,7,36 1,7 > gpurun_out/cs65.log 2>&1; cat gpurun_out/cs65.log
LRS_WCONV_DEBUG=1 python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
LRS_CORE_IPT=2 LRS_CORE_TH=7 LRS_CORE_GRID=36 timeout 120 python tools/ctrace.py c2_bf16 > gpurun_out/ctrace65.log 2>&1; cat gpurun_out/ctrace65.log
python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
