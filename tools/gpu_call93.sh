run() { env "$@" timeout 300 python bench.py --config c2_bf16 --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b93.json 2> gpurun_out/b93.err; echo "$* : $(tail -1 gpurun_out/b93.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,2))' 2>&1 | tail -1) | $(grep 'wconv plan' gpurun_out/b93.err | head -1 | cut -c1-90)"; }
run LRS_VERBOSE=1
run LRS_VERBOSE=1 LRS_WCONV_BPI=2
run LRS_VERBOSE=1 LRS_WCONV_NS=3
run LRS_VERBOSE=1 LRS_WCONV_ERING=1
run LRS_VERBOSE=1 LRS_WCONV_TH=1
run LRS_VERBOSE=1 LRS_WCONV_CB=2
