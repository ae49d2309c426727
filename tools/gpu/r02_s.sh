mkdir -p gpurun_out/r02s; O=gpurun_out/r02s
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "gpu rc=$?" > $O/rc.txt
for c in c3 c2_bf16 c4; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 10 --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
done
timeout 2400 python tools/f2_speed_bound.py > $O/f2.log 2>&1; echo "f2 rc=$?" >> $O/rc.txt
cp profiles/r02_f2_speed_bound.json $O/ 2>/dev/null
cat $O/rc.txt; tail -2 $O/pytest_gpu.log; tail -12 $O/f2.log
