mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cp.py tests/test_gpu_core_fused.py tests/test_gpu_parity.py -q > gpurun_out/t76.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/t76.log; grep -E "FAILED" gpurun_out/t76.log | head
for c in c2_cp c2_bf16; do
timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b76.json 2> gpurun_out/b76.err; echo "$c $(tail -1 gpurun_out/b76.json | cut -c150-200)"
done
