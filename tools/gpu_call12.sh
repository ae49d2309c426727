mkdir -p gpurun_out; rm -f gpurun_out/rc12.txt
LRS_VERBOSE=1 timeout 300 python tools/gpu_debug.py c2_bf16 > gpurun_out/dbg_c2.log 2>&1; echo "dbg c2 rc=$?" >> gpurun_out/rc12.txt
timeout 900 python -m pytest tests/test_gpu_core_fused.py -q -x > gpurun_out/pytest_core.log 2>&1; echo "pytest core rc=$?" >> gpurun_out/rc12.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest all rc=$?" >> gpurun_out/rc12.txt
for c in c2_bf16 c3 c2_f32; do
  LRS_VERBOSE=1 timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/rc12.txt
done
cat gpurun_out/rc12.txt
