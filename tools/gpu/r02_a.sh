# round 2, call A: full GPU suite, extra peaks, default bench (C3) + C2/C4
mkdir -p gpurun_out/r02a; O=gpurun_out/r02a; rm -f $O/rc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 300 python tools/measure_extra_peaks.py > $O/peaks.log 2>&1; echo "peaks rc=$?" >> $O/rc.txt
cp profiles/measured_peaks_extra.json $O/ 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
for c in c3 c2_bf16 c4; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 10 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
done
cat $O/rc.txt
