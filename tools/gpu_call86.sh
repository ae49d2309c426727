for i in 1 2; do for c in c2_bf16 c4; do
timeout 300 python bench.py --config $c --steps 400 --warmup 10 --no-e2e --no-cpu > gpurun_out/b86.json 2> gpurun_out/b86.err; echo "$c $(tail -1 gpurun_out/b86.json | cut -c150-200)"
done; done
