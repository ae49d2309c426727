mkdir -p gpurun_out; rm -f gpurun_out/rc22.txt
timeout 900 python -m pytest tests/test_gpu_cp.py -q -x > gpurun_out/pytest_cp.log 2>&1; echo "pytest cp rc=$?" >> gpurun_out/rc22.txt
for c in c2_cp c1_cp; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/rc22.txt
done
timeout 300 python bench.py --config c2_cp --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2_cp.json 2>&1; echo "ref rc=$?" >> gpurun_out/rc22.txt
cat gpurun_out/rc22.txt
