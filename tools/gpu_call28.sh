mkdir -p gpurun_out; rm -f gpurun_out/rc28.txt
timeout 900 python -m pytest tests/test_gpu_tiny_f32.py tests/test_gpu_spadd_f32.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_28.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc28.txt
for c in c1 c2_f32; do
  r=$(LRS_VERBOSE=1 timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e 2>gpurun_out/b28.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['value']), d['roofline']['stage_us'])")
  echo "$c $r $(grep tiny gpurun_out/b28.err)" >> gpurun_out/rc28.txt
done
cat gpurun_out/rc28.txt
