mkdir -p gpurun_out; rm -f gpurun_out/rc38.txt
for c in c2_bf16 c3; do
 for env in "" "LRS_WCONV_CB=2" "LRS_WCONV_CB=2 LRS_WCONV_TH=4" "LRS_WCONV_CB=2 LRS_WCONV_TH=3"; do
  r=$(env $env LRS_VERBOSE=1 timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e 2>gpurun_out/b38.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2))")
  echo "$c [$env] $r $(grep 'wconv plan' gpurun_out/b38.err | head -1)" >> gpurun_out/rc38.txt
 done
done
cat gpurun_out/rc38.txt
