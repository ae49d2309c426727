timeout 900 python -m pytest tests/test_gpu_core_fused.py tests/test_gpu_parity.py -q > gpurun_out/t87.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t87.log
for i in 1 2; do for c in c2_bf16 c4; do
timeout 300 python bench.py --config $c --steps 400 --warmup 10 --no-e2e --no-cpu > gpurun_out/b87.json 2> gpurun_out/b87.err; echo "$c $(tail -1 gpurun_out/b87.json | cut -c150-200)"
done; done
