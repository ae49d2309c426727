# round 2 final evidence set: GPU suite, smoke, every bench line (forward C1-C5 + CP, reference arm,
# backward C3/C2/C4, decomposition C3/C2/16 layers), ncu launch lists and full captures of the dominant
# kernels -- the reports are summarised ON THE BOX and deleted (64 MiB copy-back limit)
mkdir -p gpurun_out/r02f; O=gpurun_out/r02f; rm -f $O/rc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?" >> $O/rc.txt
for c in c2_bf16 c4 c2_f32 c1 c2_cp c1_cp c5; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 10 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
done
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?" >> $O/rc.txt
for c in c3 c2_bf16 c4; do
  timeout 900 python bench.py --backward --config $c --steps 100 --warmup 10 > $O/bench_bwd_$c.json 2> $O/bench_bwd_$c.err; echo "bench bwd $c rc=$?" >> $O/rc.txt
done
for c in c3 c2_bf16 c5; do
  timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench dec $c rc=$?" >> $O/rc.txt
done
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-dense > $O/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
   python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-dense > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
timeout 120 python tools/run_bwd.py c3 3 > $O/plain_bwd.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bwd_c3.csv python tools/run_bwd.py c3 3 > $O/ncu_lb.log 2>&1; echo "ncu launches bwd rc=$?" >> $O/rc.txt
summ() {  # $1 report stem
  python tools/ncu_sum.py $O/prof_$1.ncu-rep > $O/sum_$1.txt 2>&1
  python tools/ncu_src.py $O/prof_$1.ncu-rep 25 > $O/sass_$1.txt 2>&1
}
for ck in c3:wconv c2_bf16:wconv c4:lrs_pw c2_f32:spadd c1:tiny c3:core_kernel; do
  cfg=${ck%%:*}; k=${ck##*:}; kn=${k#lrs_}
  timeout 120 python tools/run_layer.py $cfg 4 > $O/plain_$cfg.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/prof_${kn}_$cfg -f python tools/run_layer.py $cfg 4 > $O/ncu_${kn}_$cfg.log 2>&1; echo "ncu $k $cfg rc=$?" >> $O/rc.txt
  summ ${kn}_$cfg
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wgrad_kernel -s 1 -c 1 -o $O/prof_wgrad_c3 -f python tools/run_bwd.py c3 3 > $O/ncu_wgrad.log 2>&1; echo "ncu wgrad rc=$?" >> $O/rc.txt
summ wgrad_c3
timeout 300 python bench.py --decompose --config c3 --steps 2 --warmup 1 --no-cpu --no-e2e > $O/plain_dec.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp01q -s 4 -c 1 -o $O/prof_mttkrp_c3 -f python bench.py --decompose --config c3 --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_mttkrp.log 2>&1; echo "ncu mttkrp rc=$?" >> $O/rc.txt
summ mttkrp_c3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sym_pinv -s 5 -c 1 -o $O/prof_pinv_c3 -f python bench.py --decompose --config c3 --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_pinv.log 2>&1; echo "ncu pinv rc=$?" >> $O/rc.txt
summ pinv_c3
python tools/ncu_traffic.py $O > $O/ncu_traffic.log 2>&1; cp profiles/ncu_traffic.json $O/ncu_traffic.json
rm -f $O/*.ncu-rep
du -sh $O >> $O/rc.txt
cat $O/rc.txt
