mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_core_fused.py tests/test_gpu_cp.py tests/test_gpu_parity.py -q -x > gpurun_out/t82.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/t82.log; grep -E "FAILED" gpurun_out/t82.log | head
for c in c2_bf16 c3 c2_cp; do
LRS_VERBOSE=1 timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b82.json 2> gpurun_out/b82.err; echo "$c $(tail -1 gpurun_out/b82.json | cut -c150-200)"; grep autotune gpurun_out/b82.err | sort -t: -k2 -n | head -4
done
LRS_WCONV_DEBUG=1 python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
LRS_CORE_IPT=2 LRS_CORE_TH=7 LRS_CORE_GRID=36 timeout 120 python tools/ctrace.py c2_bf16 > gpurun_out/ctrace82.log 2>&1; cat gpurun_out/ctrace82.log
python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
