mkdir -p gpurun_out; rm -f gpurun_out/rcf.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rcf.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rcf.txt
for c in c2_bf16 c3 c4 c2_f32 c1 c2_cp c1_cp c5; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/rcf.txt
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2>&1; echo "ref rc=$?" >> gpurun_out/rcf.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
   python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/rcf.txt
timeout 120 python tools/gpu_debug.py c2_bf16 > gpurun_out/plain_c2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wconv -s 2 -c 1 -o gpurun_out/prof_wconv_c2 python tools/gpu_debug.py c2_bf16 > gpurun_out/ncu_c2.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/rcf.txt
cat gpurun_out/rcf.txt
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench default rc=$?" >> gpurun_out/rcf.txt
for c in c2_f32:spadd c1:tiny c2_bf16:core_kernel c4:wconv c3:wconv; do
  cfg=${c%%:*}; k=${c##*:}
  timeout 120 python tools/gpu_debug.py $cfg > gpurun_out/plain_$cfg.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_${k}_$cfg -f python tools/gpu_debug.py $cfg > gpurun_out/ncu_${k}_$cfg.log 2>&1; echo "ncu $k $cfg rc=$?" >> gpurun_out/rcf.txt
done
cat gpurun_out/rcf.txt
timeout 1500 python tools/f2_speed_bound.py > gpurun_out/f2.log 2>&1; echo "f2 rc=$?" >> gpurun_out/rcf.txt
cat gpurun_out/rcf.txt
