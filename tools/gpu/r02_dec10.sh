# decomposition (f4): certified Cholesky path for the pseudo-inverse: tests, probe (both paths), bench
mkdir -p gpurun_out/dec10; O=gpurun_out/dec10; rm -f $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x > $O/pytest_dec.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
./tools/pinv_probe 128 0 > $O/pinv_probe.log 2>&1; ./tools/pinv_probe 128 1 >> $O/pinv_probe.log 2>&1
for c in c3 c2_bf16 c5; do
  timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
done
python tools/decomp_det.py c2_decomp > $O/decomp_det.log 2>&1
cat $O/rc.txt
