mkdir -p gpurun_out
run() { env "$@" timeout 300 python bench.py --config c4 --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/b68.json 2> gpurun_out/b68.err; echo "$* : $(tail -1 gpurun_out/b68.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,2))') | $(grep 'wconv plan' gpurun_out/b68.err | head -1)"; }
run LRS_VERBOSE=1
run LRS_VERBOSE=1 LRS_WCONV_REUSE=1
run LRS_VERBOSE=1 LRS_WCONV_REUSE=1 LRS_WCONV_TH=2
run LRS_VERBOSE=1 LRS_WCONV_REUSE=1 LRS_WCONV_NS=3
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "c4 or svd or 1x1" > gpurun_out/t68.log 2>&1; tail -1 gpurun_out/t68.log
LRS_WCONV_REUSE=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_tc.py -q > gpurun_out/t68r.log 2>&1; tail -1 gpurun_out/t68r.log
