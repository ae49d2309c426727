mkdir -p gpurun_out; rm -f gpurun_out/rc39.txt
LRS_CORE_SEP=1 timeout 600 python -m pytest tests/test_gpu_core_fused.py -q -x > gpurun_out/pytest_39.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc39.txt
for c in c2_bf16 c3; do
 for env in "" "LRS_CORE_SEP=1"; do
  r=$(env $env timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), d['roofline']['stage_us'])")
  echo "$c [$env] $r" >> gpurun_out/rc39.txt
 done
done
cat gpurun_out/rc39.txt
