# backward pass side-stream recompute: tests, bench C3 / C2 / C4, launch list
mkdir -p gpurun_out/bwd7; O=gpurun_out/bwd7; rm -f $O/rc.txt
timeout 1200 python -m pytest tests/test_gpu_backward.py -q -x > $O/pytest_bwd.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for c in c3 c2_bf16 c4; do
  LRS_VERBOSE= timeout 900 python bench.py --backward --config $c --steps 50 --warmup 5 --no-cpu > $O/bench_bwd_$c.json 2> $O/bench_bwd_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
done
LRS_VERBOSE=1 timeout 120 python tools/run_bwd.py c3 3 > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bwd_c3.csv python tools/run_bwd.py c3 3 > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
cat $O/rc.txt
