#!/bin/bash
mkdir -p gpurun_out
for c in c2_bf16 c2_f32 c3 c4 c1; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/rc.txt
done
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/rc.txt
cat gpurun_out/rc.txt
