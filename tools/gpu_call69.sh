mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiny_f32.py tests/test_gpu_parity.py tests/test_gpu_epilogue.py tests/test_gpu_cp.py -q > gpurun_out/t69.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/t69.log; grep -E "^E |FAILED" gpurun_out/t69.log | head
for cb in 0 1 2 3 4; do
LRS_TINY_CB=$cb LRS_VERBOSE=1 timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b69.json 2> gpurun_out/b69.err; echo "cb=$cb $(tail -1 gpurun_out/b69.json | cut -c150-200) $(grep tiny: gpurun_out/b69.err | head -1)"
done
