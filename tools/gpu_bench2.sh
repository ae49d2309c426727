mkdir -p gpurun_out; rm -f gpurun_out/rcb.txt
for c in c2_bf16 c3 c4 c2_f32 c1; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/rcb.txt
done
cat gpurun_out/rcb.txt
