mkdir -p gpurun_out; rm -f gpurun_out/rc13.txt
timeout 900 python -m pytest tests/test_gpu_core_fused.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_core.log 2>&1; echo "pytest core rc=$?" >> gpurun_out/rc13.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest all rc=$?" >> gpurun_out/rc13.txt
for c in c2_bf16 c3; do
  LRS_VERBOSE=1 timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/rc13.txt
  for ipt in 1 2 3; do
    r=$(LRS_CORE_IPT=$ipt timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), d['roofline']['stage_us'])")
    echo "$c ipt=$ipt $r" >> gpurun_out/rc13.txt
  done
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:core_kernel -c 1 -o gpurun_out/prof_core_$c -f python tools/gpu_debug.py $c > gpurun_out/ncu_core_$c.log 2>&1; echo "ncu $c rc=$?" >> gpurun_out/rc13.txt
done
cat gpurun_out/rc13.txt
