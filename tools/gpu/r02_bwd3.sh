# backward pass: bench C3 (fixed verify), ncu launch list and one full capture of the weight-gradient kernel
mkdir -p gpurun_out/bwd3; O=gpurun_out/bwd3; rm -f $O/rc.txt
timeout 900 python bench.py --backward --config c3 --steps 50 --warmup 5 > $O/bench_bwd_c3.json 2> $O/bench_bwd_c3.err; echo "bench rc=$?" >> $O/rc.txt
timeout 120 python tools/run_bwd.py c3 3 > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bwd_c3.csv python tools/run_bwd.py c3 3 > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wgrad_kernel -s 1 -c 1 -o $O/prof_wgrad_c3 -f python tools/run_bwd.py c3 3 > $O/ncu_w.log 2>&1; echo "ncu wgrad rc=$?" >> $O/rc.txt
cat $O/rc.txt
