timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_tc.py tests/test_gpu_epilogue.py tests/test_gpu_core_fused.py -q > gpurun_out/t92.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t92.log; grep FAILED gpurun_out/t92.log | head -5
for e in X=1 LRS_NO_TMA_Y=1; do for c in c2_bf16 c3 c4; do
env $e timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', '$c', round(d['ms_per_step']*1e3,2))"
done; done
