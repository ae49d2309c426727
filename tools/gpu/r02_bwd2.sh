# backward pass: GPU tests, bench lines (C3 / C2 / C4 backward)
mkdir -p gpurun_out/bwd2; O=gpurun_out/bwd2; rm -f $O/rc.txt
timeout 1200 python -m pytest tests/test_gpu_backward.py -q > $O/pytest_bwd.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for c in c3 c2_bf16 c4; do
  LRS_VERBOSE= timeout 900 python bench.py --backward --config $c --steps 50 --warmup 5 > $O/bench_bwd_$c.json 2> $O/bench_bwd_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
done
cat $O/rc.txt
