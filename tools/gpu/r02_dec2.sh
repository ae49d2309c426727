# decomposition (f4): bench lines (C3 / C2 weight shapes), fp64 DFMA peak, launch list
mkdir -p gpurun_out/dec2; O=gpurun_out/dec2; rm -f $O/rc.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dfma_peak tools/dfma_peak.cu && ./tools/dfma_peak > $O/dfma.json 2>&1; echo "dfma rc=$?" >> $O/rc.txt
for c in c3 c2_bf16; do
  timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_dec_c3.csv python bench.py --decompose --config c3 --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp01 -s 4 -c 1 -o $O/prof_mttkrp01_c3 -f python bench.py --decompose --config c3 --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_m.log 2>&1; echo "ncu mttkrp rc=$?" >> $O/rc.txt
cat $O/rc.txt
