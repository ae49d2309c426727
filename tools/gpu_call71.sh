mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cp.py tests/test_gpu_core_fused.py -q > gpurun_out/t71.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/t71.log; grep -E "^E |FAILED" gpurun_out/t71.log | head
LRS_VERBOSE=1 timeout 300 python bench.py --config c2_cp --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b71.json 2> gpurun_out/b71.err; echo "c2_cp $(tail -1 gpurun_out/b71.json | cut -c150-200)"; grep autotune gpurun_out/b71.err
python -c "
import json; d=json.loads(open('gpurun_out/b71.json').read().strip().splitlines()[-1]); print(d['roofline']['kernel'], d['roofline']['bound'], d['roofline']['frac'], d['roofline']['stage_us'])"
