#!/bin/bash
# round 2, last session: validate HEAD (after the pseudo-inverse LDS/STS change) on a B200
val() {
  mkdir -p gpurun_out/s3; O=gpurun_out/s3; rm -f $O/rc.txt
  timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
  timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?" >> $O/rc.txt
  timeout 600 python bench.py --decompose --steps 30 --warmup 3 > $O/bench_dec_c3.json 2> $O/bench_dec_c3.err; echo "bench dec c3 rc=$?" >> $O/rc.txt
  timeout 600 python bench.py --decompose --tucker2 --steps 30 --warmup 3 > $O/bench_dec_t2.json 2> $O/bench_dec_t2.err; echo "bench dec t2 rc=$?" >> $O/rc.txt
  for c in c4 c2_f32; do
    timeout 600 python bench.py --config $c --steps 200 --warmup 10 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  cat $O/rc.txt
}

db() {
  # the double-buffered fp32 sparse/expansion kernel: whole GPU suite, then the C2-fp32 line
  mkdir -p gpurun_out/db; O=gpurun_out/db; rm -f $O/rc.txt
  LRS_VERBOSE=1 timeout 300 python bench.py --config c2_f32 --steps 200 --warmup 10 > $O/bench_c2_f32.json 2> $O/bench_c2_f32.err; echo "bench c2_f32 rc=$?" >> $O/rc.txt
  timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}
unr() {
  # staging loops unrolled by 2 (two items' loads in flight per thread): C2-fp32 line + fp32 tests
  mkdir -p gpurun_out/unr; O=gpurun_out/unr; rm -f $O/rc.txt
  for i in 1 2; do timeout 300 python bench.py --config c2_f32 --steps 200 --warmup 10 --no-cpu > $O/bench_c2_f32_$i.json 2> $O/bench_c2_f32_$i.err; echo "bench c2_f32 rc=$?" >> $O/rc.txt; done
  timeout 900 python -m pytest tests/test_gpu_spadd_f32.py tests/test_gpu_parity.py tests/test_gpu_epilogue.py -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}
"$@"
