mkdir -p gpurun_out
echo skip-tests
tail -2 gpurun_out/t84.log; grep -E "FAILED" gpurun_out/t84.log | head
for c in c2_bf16 c3 c2_cp; do
for e in X=1 LRS_NO_FLAGS=1; do
env $e LRS_VERBOSE=1 timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b84.json 2> gpurun_out/b84.err; echo "$c $e $(tail -1 gpurun_out/b84.json | cut -c150-200)"; grep autotune gpurun_out/b84.err | sort -t: -k2 -n | head -2
done; done
