mkdir -p gpurun_out; rm -f gpurun_out/rc41.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spadd_f32.py tests/test_gpu_cp.py -q -x > gpurun_out/pytest_41.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc41.txt
for c in c2_f32 c1_cp c2_bf16; do
  r=$(timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['value']), d['roofline']['stage_us'])")
  echo "$c $r" >> gpurun_out/rc41.txt
done
cat gpurun_out/rc41.txt
