mkdir -p gpurun_out
run() { env "$@" timeout 300 python bench.py --config c4 --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/b67.json 2> gpurun_out/b67.err; echo "$* : $(tail -1 gpurun_out/b67.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,2))') | $(grep 'wconv plan' gpurun_out/b67.err | head -1)"; }
run LRS_VERBOSE=1
run LRS_VERBOSE=1 LRS_WCONV_TH=2
run LRS_VERBOSE=1 LRS_WCONV_TH=1 LRS_WCONV_CPW=2
run LRS_VERBOSE=1 LRS_WCONV_TH=1 LRS_WCONV_CPW=1
run LRS_VERBOSE=1 LRS_WCONV_REUSE=1
run LRS_VERBOSE=1 LRS_WCONV_REUSE=1 LRS_WCONV_TH=2
run LRS_VERBOSE=1 LRS_WCONV_NS=2
run LRS_VERBOSE=1 LRS_WCONV_BPI=2
run LRS_VERBOSE=1 LRS_WCONV_CB=2
