mkdir -p gpurun_out; rm -f gpurun_out/rc50.txt
timeout 900 python -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_parity.py tests/test_gpu_epilogue.py tests/test_gpu_core_fused.py -q -x > gpurun_out/pytest_50.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc50.txt
for c in c2_bf16 c3 c4; do
  r=$(timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['value']), d['roofline']['stage_us'])")
  echo "$c $r" >> gpurun_out/rc50.txt
done
cat gpurun_out/rc50.txt
