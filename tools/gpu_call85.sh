mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_core_fused.py tests/test_gpu_cp.py tests/test_gpu_parity.py -q > gpurun_out/t85.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/t85.log; grep -E "FAILED" gpurun_out/t85.log | head
LRS_FLAGS=1 timeout 600 python -m pytest tests/test_gpu_cp.py -q > gpurun_out/t85b.log 2>&1; echo "cp flags rc=$?"; tail -1 gpurun_out/t85b.log
timeout 300 python bench.py --config c2_bf16 --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b85.json 2> gpurun_out/b85.err; echo "c2 $(tail -1 gpurun_out/b85.json | cut -c150-200)"
