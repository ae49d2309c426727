mkdir -p gpurun_out; rm -f gpurun_out/skip11.log
for c in c2_bf16 c3 c4 c2_f32 c1; do for sk in 0 1 2 3 4 8 12; do
  r=$(LRS_SKIP=$sk timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2))")
  echo "$c skip=$sk step_us=$r" >> gpurun_out/skip11.log
done; done
cat gpurun_out/skip11.log
