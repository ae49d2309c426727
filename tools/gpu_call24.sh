mkdir -p gpurun_out; rm -f gpurun_out/plan24.log
for c in c4 c2_bf16 c3; do
 for env in "" "LRS_WCONV_BPI=2" "LRS_WCONV_TH=4" "LRS_WCONV_TH=4 LRS_WCONV_BPI=2" "LRS_WCONV_TH=7" "LRS_WCONV_TH=7 LRS_WCONV_BPI=2" "LRS_WCONV_TH=1"; do
  r=$(env $env LRS_VERBOSE=1 timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu --no-e2e 2>gpurun_out/b24.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2))")
  echo "$c [$env] step_us=$r $(grep 'wconv plan' gpurun_out/b24.err)" >> gpurun_out/plan24.log
 done
done
cat gpurun_out/plan24.log
