mkdir -p gpurun_out
run() { env "$@" timeout 300 python bench.py --config c3 --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/b79.json 2> gpurun_out/b79.err; echo "$* : $(tail -1 gpurun_out/b79.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,2))' 2>&1 | tail -1) | $(grep 'wconv plan' gpurun_out/b79.err | head -1)"; }
run LRS_VERBOSE=1
run LRS_VERBOSE=1 LRS_WCONV_NWB1=1
run LRS_VERBOSE=1 LRS_WCONV_NWB1=1 LRS_WCONV_ERING=1
run LRS_VERBOSE=1 LRS_WCONV_ERING=1
LRS_WCONV_NWB1=1 LRS_WCONV_ERING=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_tc.py -q -x > gpurun_out/t79.log 2>&1; tail -1 gpurun_out/t79.log
