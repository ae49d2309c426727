timeout 600 python -m pytest tests/test_gpu_core_fused.py tests/test_gpu_cp.py -q > gpurun_out/t90.log 2>&1; echo rc=$?; tail -1 gpurun_out/t90.log
for d in 0 8; do for c in c2_bf16 c3 c2_cp; do
LRS_CORE_DBG=$d timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg=$d', '$c', round(d['ms_per_step']*1e3,2))"
done; done
