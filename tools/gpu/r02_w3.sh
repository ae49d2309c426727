# round 2, call W3: evidence set (final code) -- GPU suite, smoke, every bench line, reference arm, ncu launch list + full
# captures; the ncu reports are summarised on the box (tools/ncu_sum.py / ncu_src.py / ncu_traffic.py) and deleted,
# so gpurun_out/ stays under the 64 MiB copy-back limit
mkdir -p gpurun_out/r02w3; O=gpurun_out/r02w3; rm -f $O/rc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?" >> $O/rc.txt
for c in c2_bf16 c4 c2_f32 c1 c2_cp c1_cp c5; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 10 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
done
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?" >> $O/rc.txt
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-dense > $O/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
   python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-dense > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
for ck in c3:wconv c2_bf16:wconv c4:lrs_pw c2_f32:spadd c1:tiny c3:core_kernel; do
  cfg=${ck%%:*}; k=${ck##*:}; kn=${k#lrs_}
  timeout 120 python tools/run_layer.py $cfg 4 > $O/plain_$cfg.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/prof_${kn}_$cfg -f python tools/run_layer.py $cfg 4 > $O/ncu_${kn}_$cfg.log 2>&1; echo "ncu $k $cfg rc=$?" >> $O/rc.txt
  python tools/ncu_sum.py $O/prof_${kn}_$cfg.ncu-rep > $O/sum_${kn}_$cfg.txt 2>&1
  python tools/ncu_src.py $O/prof_${kn}_$cfg.ncu-rep 25 > $O/sass_${kn}_$cfg.txt 2>&1
done
python tools/ncu_traffic.py $O > $O/ncu_traffic.log 2>&1; cp profiles/ncu_traffic.json $O/ncu_traffic.json
rm -f $O/*.ncu-rep
cat $O/rc.txt
