mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cp.py tests/test_gpu_tiny_f32.py tests/test_gpu_epilogue.py -q > gpurun_out/t70.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/t70.log; grep -E "^E |FAILED" gpurun_out/t70.log | head
for c in c1_cp c1; do
LRS_VERBOSE=1 timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b70.json 2> gpurun_out/b70.err; echo "$c $(tail -1 gpurun_out/b70.json | cut -c150-200) $(grep tiny: gpurun_out/b70.err | head -1)"
done
