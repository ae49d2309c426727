mkdir -p gpurun_out
LRS_NO_AUTOTUNE=1 timeout 60 python tools/cp_debug.py > gpurun_out/cp75.log 2>&1; echo "rc=$? $(tail -1 gpurun_out/cp75.log)"
timeout 900 python -m pytest tests/test_gpu_cp.py tests/test_gpu_core_fused.py -q > gpurun_out/t75.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/t75.log; grep -E "^E |FAILED" gpurun_out/t75.log | head
LRS_VERBOSE=1 timeout 300 python bench.py --config c2_cp --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b75.json 2> gpurun_out/b75.err; echo "c2_cp $(tail -1 gpurun_out/b75.json | cut -c150-200)"; grep autotune gpurun_out/b75.err
