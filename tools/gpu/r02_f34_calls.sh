# Round 2, last session: the one-off GPU calls of the backward (f3), decomposition (f4) and
# e2e work, one shell function per call (run one: bash -c "source tools/gpu/r02_f34_calls.sh; bwd7").
# The evidence set is tools/gpu/r02_final.sh.

bwd1() {
  mkdir -p gpurun_out/bwd1; O=gpurun_out/bwd1
  LRS_VERBOSE=1 timeout 900 python -m pytest tests/test_gpu_backward.py -x -q -k "small_3x3 and matches" > $O/t1.log 2>&1; echo "t1 rc=$?" >> $O/rc.txt
  timeout 1200 python -m pytest tests/test_gpu_backward.py -q > $O/all.log 2>&1; echo "all rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}

bwd2() {
  # backward pass: GPU tests, bench lines (C3 / C2 / C4 backward)
  mkdir -p gpurun_out/bwd2; O=gpurun_out/bwd2; rm -f $O/rc.txt
  timeout 1200 python -m pytest tests/test_gpu_backward.py -q > $O/pytest_bwd.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16 c4; do
    LRS_VERBOSE= timeout 900 python bench.py --backward --config $c --steps 50 --warmup 5 > $O/bench_bwd_$c.json 2> $O/bench_bwd_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  cat $O/rc.txt
}

bwd3() {
  # backward pass: bench C3 (fixed verify), ncu launch list and one full capture of the weight-gradient kernel
  mkdir -p gpurun_out/bwd3; O=gpurun_out/bwd3; rm -f $O/rc.txt
  timeout 900 python bench.py --backward --config c3 --steps 50 --warmup 5 > $O/bench_bwd_c3.json 2> $O/bench_bwd_c3.err; echo "bench rc=$?" >> $O/rc.txt
  timeout 120 python tools/run_bwd.py c3 3 > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/rc.txt
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bwd_c3.csv python tools/run_bwd.py c3 3 > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:wgrad_kernel -s 1 -c 1 -o $O/prof_wgrad_c3 -f python tools/run_bwd.py c3 3 > $O/ncu_w.log 2>&1; echo "ncu wgrad rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}

bwd4() {
  # backward pass combined call: tests, bench C3 / C2 / C4, launch list
  mkdir -p gpurun_out/bwd5; O=gpurun_out/bwd4; rm -f $O/rc.txt
  timeout 1200 python -m pytest tests/test_gpu_backward.py -q -x > $O/pytest_bwd.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16 c4; do
    LRS_VERBOSE= timeout 900 python bench.py --backward --config $c --steps 50 --warmup 5 --no-cpu > $O/bench_bwd_$c.json 2> $O/bench_bwd_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  LRS_VERBOSE=1 timeout 120 python tools/run_bwd.py c3 3 > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/rc.txt
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bwd_c3.csv python tools/run_bwd.py c3 3 > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}

bwd5() {
  # backward pass combined call: tests, bench C3 / C2 / C4, launch list
  mkdir -p gpurun_out/bwd5; O=gpurun_out/bwd5; rm -f $O/rc.txt
  timeout 1200 python -m pytest tests/test_gpu_backward.py -q -x > $O/pytest_bwd.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16 c4; do
    LRS_VERBOSE= timeout 900 python bench.py --backward --config $c --steps 50 --warmup 5 --no-cpu > $O/bench_bwd_$c.json 2> $O/bench_bwd_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  LRS_VERBOSE=1 timeout 120 python tools/run_bwd.py c3 3 > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/rc.txt
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bwd_c3.csv python tools/run_bwd.py c3 3 > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}

bwd6() {
  # backward pass split granularity chooser: tests, bench C3 / C2 / C4, launch list
  mkdir -p gpurun_out/bwd6; O=gpurun_out/bwd6; rm -f $O/rc.txt
  timeout 1200 python -m pytest tests/test_gpu_backward.py -q -x > $O/pytest_bwd.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16 c4; do
    LRS_VERBOSE= timeout 900 python bench.py --backward --config $c --steps 50 --warmup 5 --no-cpu > $O/bench_bwd_$c.json 2> $O/bench_bwd_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  LRS_VERBOSE=1 timeout 120 python tools/run_bwd.py c3 3 > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/rc.txt
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bwd_c3.csv python tools/run_bwd.py c3 3 > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}

bwd7() {
  # backward pass side-stream recompute: tests, bench C3 / C2 / C4, launch list
  mkdir -p gpurun_out/bwd7; O=gpurun_out/bwd7; rm -f $O/rc.txt
  timeout 1200 python -m pytest tests/test_gpu_backward.py -q -x > $O/pytest_bwd.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16 c4; do
    LRS_VERBOSE= timeout 900 python bench.py --backward --config $c --steps 50 --warmup 5 --no-cpu > $O/bench_bwd_$c.json 2> $O/bench_bwd_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  LRS_VERBOSE=1 timeout 120 python tools/run_bwd.py c3 3 > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/rc.txt
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bwd_c3.csv python tools/run_bwd.py c3 3 > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}

dec1() {
  # decomposition (f4): GPU tests
  mkdir -p gpurun_out/dec1; O=gpurun_out/dec1; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x > $O/pytest_dec.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}

dec2() {
  # decomposition (f4): bench lines (C3 / C2 weight shapes), fp64 DFMA peak, launch list
  mkdir -p gpurun_out/dec2; O=gpurun_out/dec2; rm -f $O/rc.txt
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dfma_peak tools/dfma_peak.cu && ./tools/dfma_peak > $O/dfma.json 2>&1; echo "dfma rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16; do
    timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_dec_c3.csv python bench.py --decompose --config c3 --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_l.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp01 -s 4 -c 1 -o $O/prof_mttkrp01_c3 -f python bench.py --decompose --config c3 --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_m.log 2>&1; echo "ncu mttkrp rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}

dec3() {
  # decomposition (f4): tests + bench after the Jacobi fix
  mkdir -p gpurun_out/dec3; O=gpurun_out/dec3; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x > $O/pytest_dec.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16; do
    timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  cat $O/rc.txt
}

dec4() {
  # decomposition (f4): tests + bench Jacobi off-norm criterion, register-blocked MTTKRP
  mkdir -p gpurun_out/dec5; O=gpurun_out/dec5; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x > $O/pytest_dec.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16; do
    timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  cat $O/rc.txt
}

dec5() {
  # decomposition (f4): tests + bench Jacobi off-norm criterion, register-blocked MTTKRP
  mkdir -p gpurun_out/dec6; O=gpurun_out/dec6; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x > $O/pytest_dec.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16; do
    timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  cat $O/rc.txt
}

dec6() {
  # decomposition (f4): tests + bench Jacobi off-norm criterion, register-blocked MTTKRP
  mkdir -p gpurun_out/dec7; O=gpurun_out/dec7; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x > $O/pytest_dec.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16; do
    timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  cat $O/rc.txt
}

dec7() {
  # decomposition (f4): tests + bench Jacobi off-norm criterion, register-blocked MTTKRP
  mkdir -p gpurun_out/dec8; O=gpurun_out/dec8; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x > $O/pytest_dec.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16; do
    timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  cat $O/rc.txt
  ./tools/pinv_probe 128 > $O/pinv_probe.log 2>&1
}

dec8() {
  # decomposition (f4): tests + bench Jacobi off-norm criterion, register-blocked MTTKRP
  mkdir -p gpurun_out/dec8; O=gpurun_out/dec8; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x > $O/pytest_dec.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16; do
    timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  cat $O/rc.txt
  ./tools/pinv_probe 128 > $O/pinv_probe.log 2>&1
  python tools/decomp_det.py c2_decomp > $O/decomp_det.log 2>&1
}

dec9() {
  # decomposition (f4): warm-started, batched-load Jacobi: tests, probe, bench C3 / C2 / the 16 ResNet-50 weights
  mkdir -p gpurun_out/dec9; O=gpurun_out/dec9; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x > $O/pytest_dec.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  ./tools/pinv_probe 128 > $O/pinv_probe.log 2>&1
  for c in c3 c2_bf16 c5; do
    timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  python tools/decomp_det.py c2_decomp > $O/decomp_det.log 2>&1
  cat $O/rc.txt
}

dec10() {
  # decomposition (f4): certified Cholesky path for the pseudo-inverse: tests, probe (both paths), bench
  mkdir -p gpurun_out/dec10; O=gpurun_out/dec10; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x > $O/pytest_dec.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  ./tools/pinv_probe 128 0 > $O/pinv_probe.log 2>&1; ./tools/pinv_probe 128 1 >> $O/pinv_probe.log 2>&1
  for c in c3 c2_bf16 c5; do
    timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  python tools/decomp_det.py c2_decomp > $O/decomp_det.log 2>&1
  cat $O/rc.txt
}

e2e() {
  # streaming host-buffer forward: parity tests, e2e of the default bench and C2 / C4
  mkdir -p gpurun_out/e2e; O=gpurun_out/e2e; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "host_io" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  timeout 600 python bench.py --no-cpu > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?" >> $O/rc.txt
  for c in c2_bf16 c4; do
    timeout 600 python bench.py --config $c --steps 200 --warmup 10 --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  cat $O/rc.txt
}
dec11() {
  # decomposition (f4): blocked Cholesky pseudo-inverse + staged MTTKRP rows: tests, probe, bench
  mkdir -p gpurun_out/dec11; O=gpurun_out/dec11; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x > $O/pytest_dec.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  ./tools/pinv_probe 128 0 > $O/pinv_probe.log 2>&1; ./tools/pinv_probe 33 0 >> $O/pinv_probe.log 2>&1
  for c in c3 c2_bf16 c5; do
    timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  python tools/decomp_det.py c2_decomp > $O/decomp_det.log 2>&1
  cat $O/rc.txt
}

dec12() {
  # decomposition (f4): blocked Cholesky pseudo-inverse + staged MTTKRP rows: tests, probe, bench
  mkdir -p gpurun_out/dec12; O=gpurun_out/dec12; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x > $O/pytest_dec.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  ./tools/pinv_probe 128 0 > $O/pinv_probe.log 2>&1; ./tools/pinv_probe 33 0 >> $O/pinv_probe.log 2>&1
  for c in c3 c2_bf16 c5; do
    timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  python tools/decomp_det.py c2_decomp > $O/decomp_det.log 2>&1
  cat $O/rc.txt
}
refresh() {
  # final refresh after the side-stream backward and the decomposition changes: GPU suite, smoke,
  # default bench, backward and decomposition lines, the wgrad / MTTKRP / pseudo-inverse captures
  mkdir -p gpurun_out/r02g; O=gpurun_out/r02g; rm -f $O/rc.txt
  timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
  timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16 c4; do
    timeout 900 python bench.py --backward --config $c --steps 100 --warmup 10 > $O/bench_bwd_$c.json 2> $O/bench_bwd_$c.err; echo "bench bwd $c rc=$?" >> $O/rc.txt
  done
  for c in c3 c2_bf16 c5; do
    timeout 900 python bench.py --decompose --config $c --steps 30 --warmup 3 > $O/bench_dec_$c.json 2> $O/bench_dec_$c.err; echo "bench dec $c rc=$?" >> $O/rc.txt
  done
  timeout 120 python tools/run_bwd.py c3 3 > $O/plain_bwd.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bwd_c3.csv python tools/run_bwd.py c3 3 > $O/ncu_lb.log 2>&1; echo "ncu launches bwd rc=$?" >> $O/rc.txt
  summ() { python tools/ncu_sum.py $O/prof_$1.ncu-rep > $O/sum_$1.txt 2>&1; python tools/ncu_src.py $O/prof_$1.ncu-rep 25 > $O/sass_$1.txt 2>&1; }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:wgrad_kernel -s 1 -c 1 -o $O/prof_wgrad_c3 -f python tools/run_bwd.py c3 3 > $O/ncu_wgrad.log 2>&1; echo "ncu wgrad rc=$?" >> $O/rc.txt
  summ wgrad_c3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp01q -s 4 -c 1 -o $O/prof_mttkrp_c3 -f python bench.py --decompose --config c3 --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_mttkrp.log 2>&1; echo "ncu mttkrp rc=$?" >> $O/rc.txt
  summ mttkrp_c3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sym_pinv -s 5 -c 1 -o $O/prof_pinv_c3 -f python bench.py --decompose --config c3 --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_pinv.log 2>&1; echo "ncu pinv rc=$?" >> $O/rc.txt
  summ pinv_c3
  rm -f $O/*.ncu-rep
  cat $O/rc.txt
}
f32stage() {
  # fp32 kernel: coalesced X window staging -- fp32 parity tests and the C2-fp32 bench line
  mkdir -p gpurun_out/f32; O=gpurun_out/f32; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_spadd_f32.py tests/test_gpu_parity.py tests/test_gpu_bounds.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  timeout 600 python bench.py --config c2_f32 --steps 200 --warmup 10 > $O/bench_c2_f32.json 2> $O/bench_c2_f32.err; echo "bench rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}
wpair() {
  # backward: the weight-gradient kernel's CTA-pair form -- backward tests, bench C3/C2/C4 (pair and LRS_WGRAD_NO_PAIR in a tool)
  mkdir -p gpurun_out/wpair; O=gpurun_out/wpair; rm -f $O/rc.txt
  LRS_VERBOSE=1 timeout 300 python tools/run_bwd.py c3 3 > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/rc.txt
  timeout 1200 python -m pytest tests/test_gpu_backward.py -q -x > $O/pytest_bwd.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16 c4; do
    timeout 900 python bench.py --backward --config $c --steps 50 --warmup 5 --no-cpu > $O/bench_bwd_$c.json 2> $O/bench_bwd_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  cat $O/rc.txt
}

wpair2() {
  # backward: ONE padded CTA-pair weight-gradient launch -- backward tests, bench C3/C2/C4 (pair and LRS_WGRAD_NO_PAIR in a tool)
  mkdir -p gpurun_out/wpair2; O=gpurun_out/wpair2; rm -f $O/rc.txt
  LRS_VERBOSE=1 timeout 300 python tools/run_bwd.py c3 3 > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/rc.txt
  timeout 1200 python -m pytest tests/test_gpu_backward.py -q -x > $O/pytest_bwd.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16 c4; do
    timeout 900 python bench.py --backward --config $c --steps 50 --warmup 5 --no-cpu > $O/bench_bwd_$c.json 2> $O/bench_bwd_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  cat $O/rc.txt
}

wsolo() {
  # backward: the default one-CTA weight-gradient form after the pair refactor -- backward tests, bench C3/C2/C4 (pair and LRS_WGRAD_NO_PAIR in a tool)
  mkdir -p gpurun_out/wsolo; O=gpurun_out/wsolo; rm -f $O/rc.txt
  LRS_VERBOSE=1 timeout 300 python tools/run_bwd.py c3 3 > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/rc.txt
  timeout 1200 python -m pytest tests/test_gpu_backward.py -q -x > $O/pytest_bwd.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16 c4; do
    timeout 900 python bench.py --backward --config $c --steps 50 --warmup 5 --no-cpu > $O/bench_bwd_$c.json 2> $O/bench_bwd_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  cat $O/rc.txt
}
bwdedge() {
  # backward: off-grid channel counts / ranks and a 7x7 kernel
  mkdir -p gpurun_out/bwdedge; O=gpurun_out/bwdedge; rm -f $O/rc.txt
  timeout 900 python -m pytest tests/test_gpu_backward.py -q -k "odd or k7" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}
wbn() {
  # backward: weight-gradient N-tile cap (LRS_WGRAD_BN) vs the default
  mkdir -p gpurun_out/wbn; O=gpurun_out/wbn
  for c in c3 c2_bf16 c4; do
    python tools/bwd_time.py $c >> $O/log.txt 2>&1
    LRS_WGRAD_BN=128 python tools/bwd_time.py $c >> $O/log.txt 2>&1
    LRS_WGRAD_BN=192 python tools/bwd_time.py $c >> $O/log.txt 2>&1
  done
}
bwds2() {
  # backward at stride 2 (zero insertion + strided TMA boxes): the backward suite
  mkdir -p gpurun_out/bwds2; O=gpurun_out/bwds2; rm -f $O/rc.txt
  timeout 1200 python -m pytest tests/test_gpu_backward.py -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}
bwdcp() {
  # backward of the paper's CP layer (Tucker-2 embedding + dB / dC fold) and the whole backward suite
  mkdir -p gpurun_out/bwdcp; O=gpurun_out/bwdcp; rm -f $O/rc.txt
  timeout 1500 python -m pytest tests/test_gpu_backward.py -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}
final() {
  # last validation of the round: the whole GPU suite, smoke, the default bench line, the
  # Tucker-2 decomposition line and a full capture of its mode-product GEMM
  mkdir -p gpurun_out/fin; O=gpurun_out/fin; rm -f $O/rc.txt
  timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
  timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?" >> $O/rc.txt
  timeout 600 python bench.py --decompose --tucker2 --steps 30 --warmup 3 > $O/bench_dec_t2.json 2> $O/bench_dec_t2.err; echo "bench dec t2 rc=$?" >> $O/rc.txt
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgemm -s 3 -c 1 -o $O/prof_dgemm_t2 -f python bench.py --decompose --tucker2 --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_dgemm.log 2>&1; echo "ncu dgemm rc=$?" >> $O/rc.txt
  python tools/ncu_sum.py $O/prof_dgemm_t2.ncu-rep > $O/sum_dgemm_t2.txt 2>&1
  rm -f $O/*.ncu-rep
  cat $O/rc.txt
}
