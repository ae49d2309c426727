mkdir -p gpurun_out; rm -f gpurun_out/rc26.txt
for c in c4 c2_bf16 c3; do
  r=$(timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['value']))")
  echo "$c $r" >> gpurun_out/rc26.txt
done
timeout 600 python -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2 >> gpurun_out/rc26.txt
cat gpurun_out/rc26.txt
