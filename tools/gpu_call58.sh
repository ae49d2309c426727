mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_core_fused.py tests/test_gpu_parity.py tests/test_gpu_sparse_tc.py tests/test_gpu_epilogue.py tests/test_gpu_cp.py -q > gpurun_out/t58.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/t58.log
for c in c2_bf16 c3 c4 c2_cp; do
LRS_VERBOSE=1 timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b58_$c.json 2> gpurun_out/b58_$c.err; echo "$c rc=$?"; tail -1 gpurun_out/b58_$c.json | cut -c140-200; grep "autotune" gpurun_out/b58_$c.err | head -12
done
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/b58_c5.json 2> gpurun_out/b58_c5.err; echo "c5 rc=$?"; tail -1 gpurun_out/b58_c5.json | cut -c1-200
