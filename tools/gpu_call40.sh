mkdir -p gpurun_out; rm -f gpurun_out/rc40.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_40.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc40.txt
for c in c2_bf16 c3 c4 c2_f32 c1; do
  r=$(timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), 'e2e', round(d['e2e']['value']), d['e2e']['h2d_bytes_per_step'], d['e2e']['d2h_bytes_per_step'])")
  echo "$c $r" >> gpurun_out/rc40.txt
done
cat gpurun_out/rc40.txt
