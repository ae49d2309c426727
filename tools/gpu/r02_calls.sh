# Round-2 GPU calls (one shell function per /usr/local/graft/bin/gpurun call), kept for provenance of
# the logs under profiles/: run one with  gpurun -- bash -c "source tools/gpu/r02_calls.sh; call_<id>"
# (the evidence sets are tools/gpu/r02_v.sh and tools/gpu/r02_w2.sh).

call_a() {
  # round 2, call A: full GPU suite, extra peaks, default bench (C3) + C2/C4
  mkdir -p gpurun_out/r02a; O=gpurun_out/r02a; rm -f $O/rc.txt
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
  timeout 300 python tools/measure_extra_peaks.py > $O/peaks.log 2>&1; echo "peaks rc=$?" >> $O/rc.txt
  cp profiles/measured_peaks_extra.json $O/ 2>/dev/null
  timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
  for c in c3 c2_bf16 c4; do
    timeout 600 python bench.py --config $c --steps 200 --warmup 10 > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  cat $O/rc.txt
}

call_b() {
  # round 2, call B: timing ablations (experiment build) of C3 / C4 / C2 + wconv trace of C3
  mkdir -p gpurun_out/r02b; O=gpurun_out/r02b
  LRS_EXPERIMENTS=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1 || exit 1
  for c in c3 c4 c2_bf16; do
  timeout 300 python tools/ablate.py $c base "LRS_SKIP=1" "LRS_SKIP=4" "LRS_SKIP=1 LRS_WCONV_DBG=1" "LRS_SKIP=1 LRS_WCONV_DBG=8" \
    "LRS_SKIP=1 LRS_WCONV_DBG=2" "LRS_SKIP=1 LRS_WCONV_DBG=64" "LRS_SKIP=1 LRS_WCONV_DBG=66" "LRS_SKIP=1 LRS_WCONV_DBG=16" \
    "LRS_SKIP=1 LRS_WCONV_DBG=67" "LRS_NO_PDL=1" > $O/ablate_$c.log 2>&1
  done
  LRS_WCONV_DBG=0 timeout 120 python tools/wtrace.py c3 > $O/wtrace_c3.log 2>&1
  timeout 120 python tools/wtrace.py c4 > $O/wtrace_c4.log 2>&1
  tail -n 3 $O/*.log
}

call_c() {
  # round 2, call C: timing ablations (experiment build) of C3 / C4 / C2 + core trace of C3
  mkdir -p gpurun_out/r02c; O=gpurun_out/r02c
  LRS_EXPERIMENTS=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1 || exit 1
  for c in c3 c4 c2_bf16; do
  timeout 300 python tools/ablate.py $c base "LRS_SKIP=1" "LRS_SKIP=4" "LRS_SKIP=1 LRS_WCONV_DBG=1" "LRS_SKIP=1 LRS_WCONV_DBG=8" \
    "LRS_SKIP=1 LRS_WCONV_DBG=2" "LRS_SKIP=1 LRS_WCONV_DBG=64" "LRS_SKIP=1 LRS_WCONV_DBG=66" "LRS_SKIP=1 LRS_WCONV_DBG=16" \
    "LRS_SKIP=1 LRS_WCONV_DBG=67" "LRS_NO_PDL=1" "LRS_CORE_DBG=4 LRS_SKIP=4" > $O/ablate_$c.log 2>&1
  done
  timeout 120 python tools/ctrace.py c3 > $O/ctrace_c3.log 2>&1
  LRS_VERBOSE=1 timeout 120 python tools/ablate.py c3 base > $O/verbose_c3.log 2>&1
  tail -n 15 $O/*.log
}

call_d() {
  # round 2, call D: the channel-stationary 1x1 kernel (C4)
  mkdir -p gpurun_out/r02d; O=gpurun_out/r02d
  LRS_VERBOSE=1 timeout 300 python -m pytest tests/test_gpu_pw.py -x -q > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
  timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "gpu rc=$?" >> $O/rc.txt
  timeout 300 python bench.py --config c4 --steps 200 --warmup 10 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench rc=$?" >> $O/rc.txt
  LRS_VERBOSE=1 timeout 120 python -c "
  import workloads
  from paper_2006_06443_b200 import LrsConv
  LrsConv.from_inputs(workloads.generate(workloads.CONFIGS['c4'], batch=1), batch_max=128)" > $O/plan_c4.log 2>&1
  cat $O/rc.txt
}

call_d1() {
  mkdir -p gpurun_out/r02d1; O=gpurun_out/r02d1
  timeout 600 python -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_parity.py tests/test_gpu_bench_pattern.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_EPI=scratch" "LRS_WCONV_EPI=direct" "LRS_WCONV_EPI=direct LRS_WCONV_NS=3" > $O/ablate_c3.log 2>&1
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_bf16 base "LRS_WCONV_EPI=scratch" "LRS_WCONV_EPI=direct" > $O/ablate_c2.log 2>&1
  cat $O/rc.txt; tail -3 $O/pytest.log; grep "wconv plan\|c3 \[\|c2_bf16 \[" $O/ablate_c3.log $O/ablate_c2.log
}

call_d2() {
  mkdir -p gpurun_out/r02d2; O=gpurun_out/r02d2
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_ERING=1" "LRS_WCONV_ERING=1 LRS_WCONV_EPI=direct" "LRS_WCONV_ERING=1 LRS_WCONV_EPI=direct LRS_WCONV_NS=2" > $O/ablate_c3.log 2>&1
  grep "wconv plan\|c3 \[\|rror" $O/ablate_c3.log
}

call_d3() {
  mkdir -p gpurun_out/r02d3; O=gpurun_out/r02d3
  timeout 300 python tools/ablate.py c3 base "CFG_density=0.02" "CFG_density=0.01" "CFG_density=0.0" "CFG_density=0.1" > $O/ablate_c3.log 2>&1
  timeout 300 python tools/ablate.py c2_bf16 base "CFG_density=0.02" "CFG_density=0.0" > $O/ablate_c2.log 2>&1
  cat $O/*.log | grep "\[\|rror"
}

call_e() {
  # round 2, call E: ncu of the pw kernel at C4; C3 one-block-item plans
  mkdir -p gpurun_out/r02e; O=gpurun_out/r02e
  timeout 120 python tools/run_layer.py c4 4 > $O/plain_c4.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lrs_pw -s 2 -c 1 -o $O/prof_pw_c4 -f python tools/run_layer.py c4 4 > $O/ncu_pw_c4.log 2>&1; echo "ncu rc=$?" > $O/rc.txt
  timeout 300 python tools/ablate.py c3 base "LRS_WCONV_BPI=1 LRS_WCONV_NS=6" "LRS_WCONV_BPI=1 LRS_WCONV_NS=5" "LRS_WCONV_BPI=1 LRS_WCONV_NS=4" > $O/ablate_c3.log 2>&1; echo "abl rc=$?" >> $O/rc.txt
  timeout 300 python tools/ablate.py c4 base "LRS_PW_MPC=2 LRS_PW_BP=112" "LRS_PW_MPC=2 LRS_PW_BP=96" "LRS_PW_MPC=4 LRS_PW_BP=64" "LRS_NO_PW=1" > $O/ablate_c4.log 2>&1; echo "abl4 rc=$?" >> $O/rc.txt
  cat $O/rc.txt
}

call_e1() {
  mkdir -p gpurun_out/r02e1; O=gpurun_out/r02e1
  timeout 600 python -m pytest tests/test_gpu_overlap.py -x -q > $O/pytest_overlap.log 2>&1; echo "overlap rc=$?" > $O/rc.txt
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_NO_EARLY=1" > $O/ablate_c3.log 2>&1
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_bf16 base "LRS_NO_EARLY=1" > $O/ablate_c2.log 2>&1
  timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "gpu rc=$?" >> $O/rc.txt
  cat $O/rc.txt; tail -3 $O/pytest_overlap.log; tail -3 $O/pytest_gpu.log; grep "autotune\|c3 \[\|c2_bf16 \[" $O/ablate_c3.log $O/ablate_c2.log
}

call_e2() {
  mkdir -p gpurun_out/r02e2; O=gpurun_out/r02e2
  LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
  timeout 300 python tools/wtrace.py c3 > $O/wtrace_c3.log 2>&1
  timeout 300 python tools/ctrace.py c3 > $O/ctrace_c3.log 2>&1
  cat $O/wtrace_c3.log | head -3; cat $O/ctrace_c3.log
}

call_e3() {
  mkdir -p gpurun_out/r02e3; O=gpurun_out/r02e3
  timeout 900 python -m pytest tests/test_gpu_core_fused.py tests/test_gpu_parity.py tests/test_gpu_bench_pattern.py tests/test_gpu_overlap.py tests/test_gpu_cp.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_CORE_SPLIT_RING=1" > $O/ablate_c3.log 2>&1
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_bf16 base "LRS_CORE_SPLIT_RING=1" > $O/ablate_c2.log 2>&1
  cat $O/rc.txt; tail -3 $O/pytest.log; grep "c3 \[\|c2_bf16 \[" $O/ablate_c3.log $O/ablate_c2.log; grep "core:" $O/ablate_c3.log | sort | uniq -c | head
}

call_e4() {
  mkdir -p gpurun_out/r02e4; O=gpurun_out/r02e4
  timeout 300 python tools/ablate.py c4 base > $O/ablate_c4.log 2>&1
  timeout 300 python tools/ablate.py c3 base > $O/ablate_c3.log 2>&1
  timeout 300 python tools/ablate.py c2_bf16 base > $O/ablate_c2.log 2>&1
  timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "gpu rc=$?" > $O/rc.txt
  cat $O/rc.txt; tail -3 $O/pytest_gpu.log; grep "\[" $O/ablate_c4.log $O/ablate_c3.log $O/ablate_c2.log
}

call_e5() {
  mkdir -p gpurun_out/r02e5; O=gpurun_out/r02e5
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c4 base "LRS_PW_CPI=1" "LRS_PW_CPI=2" "LRS_PW_CPI=4" > $O/ablate_c4.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_pw.py tests/test_gpu_bench_pattern.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  cat $O/rc.txt; tail -3 $O/pytest.log; grep "pw plan\|c4 \[" $O/ablate_c4.log
}

call_e6() {
  mkdir -p gpurun_out/r02e6; O=gpurun_out/r02e6
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c4 base "LRS_PW_MPC=2 LRS_PW_BP=128 LRS_PW_CPI=1" "LRS_PW_MPC=2 LRS_PW_BP=128 LRS_PW_CPI=2" "LRS_PW_MPC=1 LRS_PW_BP=128 LRS_PW_CPI=1" "LRS_PW_MPC=2 LRS_PW_BP=96 LRS_PW_CPI=2" "LRS_PW_MPC=1 LRS_PW_BP=96 LRS_PW_CPI=2" "LRS_PW_MPC=2 LRS_PW_BP=64 LRS_PW_CPI=4" > $O/ablate_c4.log 2>&1
  grep "pw plan\|c4 \[" $O/ablate_c4.log
}

call_e7() {
  mkdir -p gpurun_out/r02e7; O=gpurun_out/r02e7
  LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
  LRS_PW_MPC=2 LRS_PW_BP=96 LRS_PW_CPI=2 timeout 300 python tools/ptrace.py c4 > $O/ptrace_a.log 2>&1
  LRS_PW_MPC=2 LRS_PW_BP=96 LRS_PW_CPI=2 LRS_PW_DBG=7 timeout 300 python tools/ptrace.py c4 > $O/ptrace_dbg7.log 2>&1
  LRS_PW_MPC=2 LRS_PW_BP=96 LRS_PW_CPI=2 timeout 300 python tools/ablate.py c4 base "LRS_SKIP=1" "LRS_SKIP=1 LRS_PW_DBG=1" "LRS_SKIP=1 LRS_PW_DBG=2" "LRS_SKIP=1 LRS_PW_DBG=4" "LRS_SKIP=1 LRS_PW_DBG=7" > $O/ablate.log 2>&1
  cat $O/ptrace_a.log $O/ptrace_dbg7.log | cut -c1-600; grep "c4 \[" $O/ablate.log
}

call_e8() {
  mkdir -p gpurun_out/r02e8; O=gpurun_out/r02e8
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c4 base "LRS_PW_MPC=2 LRS_PW_BP=96 LRS_PW_CPI=2" "LRS_PW_MPC=2 LRS_PW_BP=96 LRS_PW_CPI=1" "LRS_PW_MPC=1 LRS_PW_BP=128 LRS_PW_CPI=2" "LRS_PW_MPC=2 LRS_PW_BP=64 LRS_PW_CPI=2" "LRS_PW_MPC=1 LRS_PW_BP=96 LRS_PW_CPI=2" > $O/ablate_c4.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_pw.py tests/test_gpu_epilogue.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  cat $O/rc.txt; tail -2 $O/pytest.log; grep "pw plan\|c4 \[" $O/ablate_c4.log
}

call_f() {
  # round 2, call F: pw timeline (debug build) + pw tests
  mkdir -p gpurun_out/r02f; O=gpurun_out/r02f
  timeout 300 python -m pytest tests/test_gpu_pw.py -x -q > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
  LRS_WCONV_DEBUG=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1
  LRS_VERBOSE=1 timeout 120 python tools/ptrace.py c4 > $O/ptrace_c4.log 2>&1
  LRS_PW_MPC=2 LRS_PW_BP=112 timeout 120 python tools/ptrace.py c4 > $O/ptrace_c4_m2.log 2>&1
  cat $O/rc.txt
}

call_f1() {
  mkdir -p gpurun_out/r02f1; O=gpurun_out/r02f1
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_f32 base "LRS_F32_FUSED=1" "CFG_density=0.0" "LRS_F32_FUSED=1 CFG_density=0.0" > $O/ablate.log 2>&1
  grep "c2_f32 \[" $O/ablate.log
}

call_f2() {
  mkdir -p gpurun_out/r02f2; O=gpurun_out/r02f2
  timeout 900 python -m pytest tests/test_gpu_pw.py tests/test_gpu_sparse_tc.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c4 base "LRS_NO_AUTOTUNE=1" "LRS_NO_SPTC=1" > $O/ablate_c4.log 2>&1
  timeout 300 python tools/ablate.py c2_bf16 base "LRS_NO_SPTC=1" > $O/ablate_c2.log 2>&1
  timeout 300 python tools/ablate.py c3 base "LRS_NO_SPTC=1" > $O/ablate_c3.log 2>&1
  cat $O/rc.txt; tail -2 $O/pytest.log; grep "autotune pw\|\[" $O/ablate_c4.log | grep -v "core:" ; grep "\[" $O/ablate_c2.log $O/ablate_c3.log
}

call_f3() {
  mkdir -p gpurun_out/r02f3; O=gpurun_out/r02f3
  LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
  LRS_VERBOSE=1 timeout 300 python tools/wtrace.py c2_bf16 > $O/wtrace_c2.log 2>&1
  timeout 300 python tools/ctrace.py c2_bf16 > $O/ctrace_c2.log 2>&1
  grep "plan\|core:" $O/wtrace_c2.log | tail -3; grep -v "^\[lrs\]\|plan" $O/wtrace_c2.log | cut -c1-700 | head -8; cat $O/ctrace_c2.log
}

call_f4() {
  mkdir -p gpurun_out/r02f4; O=gpurun_out/r02f4
  LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
  timeout 300 python tools/ablate.py c2_bf16 base "LRS_CORE_DBG=8" "LRS_CORE_DBG=16" "LRS_CORE_DBG=24" "LRS_CORE_DBG=4" > $O/ablate_c2.log 2>&1
  timeout 300 python tools/ablate.py c3 base "LRS_CORE_DBG=8" "LRS_CORE_DBG=16" "LRS_CORE_DBG=24" "LRS_CORE_DBG=4" > $O/ablate_c3.log 2>&1
  grep "\[" $O/ablate_c2.log $O/ablate_c3.log
}

call_f5() {
  mkdir -p gpurun_out/r02f5; O=gpurun_out/r02f5
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c4 base "LRS_A1_MB1=1" > $O/ablate_c4.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_pw.py tests/test_gpu_bench_pattern.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  cat $O/rc.txt; tail -3 $O/pytest.log; grep "c4 \[" $O/ablate_c4.log
}

call_g() {
  # round 2, call G: pw multi-lane producer
  mkdir -p gpurun_out/r02g; O=gpurun_out/r02g
  timeout 300 python -m pytest tests/test_gpu_pw.py -x -q > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
  timeout 300 python tools/ablate.py c4 base "LRS_PW_MPC=2 LRS_PW_BP=112" "LRS_PW_MPC=2 LRS_PW_BP=96" "LRS_PW_MPC=1 LRS_PW_BP=64" > $O/ablate_c4.log 2>&1; echo "abl4 rc=$?" >> $O/rc.txt
  LRS_WCONV_DEBUG=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1
  LRS_VERBOSE=1 timeout 120 python tools/ptrace.py c4 > $O/ptrace_c4.log 2>&1
  cat $O/rc.txt
}

call_g1() {
  mkdir -p gpurun_out/r02g1; O=gpurun_out/r02g1
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_GATHER=0" "LRS_WCONV_GATHER=1" > $O/ablate_c3.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_pw.py tests/test_gpu_parity.py tests/test_gpu_bench_pattern.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  cat $O/rc.txt; tail -15 $O/pytest.log; grep "wconv plan\|c3 \[\|rror" $O/ablate_c3.log
}

call_g2() {
  mkdir -p gpurun_out/r02g2; O=gpurun_out/r02g2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lrs_wconv -s 2 -c 1 -o $O/prof_wconv_c3 -f python tools/run_layer.py c3 4 > $O/ncu.log 2>&1; echo "ncu rc=$?"
  tail -3 $O/ncu.log
}

call_g3() {
  mkdir -p gpurun_out/r02g3; O=gpurun_out/r02g3
  LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
  timeout 300 python tools/wtrace.py c3 > $O/wtrace_c3.log 2>&1
  LRS_WCONV_GATHER=0 timeout 300 python tools/wtrace.py c3 > $O/wtrace_c3_res.log 2>&1
  LRS_NO_AUTOTUNE=1 timeout 300 python tools/wtrace.py c3 > $O/wtrace_c3_noat.log 2>&1
  cat $O/wtrace_c3.log | head -4; head -2 $O/wtrace_c3_res.log;  head -2 $O/wtrace_c3_noat.log
}

call_g4() {
  mkdir -p gpurun_out/r02g4; O=gpurun_out/r02g4
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_CORE_GRID=20" "LRS_CORE_GRID=40" "LRS_CORE_GRID=74" "LRS_CORE_GRID=148" > $O/ablate_c3.log 2>&1
  grep "autotune\|core plan\|c3 \[" $O/ablate_c3.log | head -40
}

call_g5() {
  mkdir -p gpurun_out/r02g5; O=gpurun_out/r02g5
  LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
  timeout 300 python tools/ctrace.py c3 > $O/ctrace_c3.log 2>&1
  LRS_CORE_IPT=1 LRS_CORE_TH=7 timeout 300 python tools/ctrace.py c3 > $O/ctrace_c3_ipt1.log 2>&1
  LRS_CORE_IPT=2 LRS_CORE_TH=7 timeout 300 python tools/ctrace.py c3 > $O/ctrace_c3_ipt2.log 2>&1
  cat $O/ctrace_c3*.log
}

call_i() {
  mkdir -p gpurun_out/r02i; O=gpurun_out/r02i
  LRS_EXPERIMENTS=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1 || exit 1
  timeout 300 python tools/ablate.py c4 base "LRS_SKIP=1" "LRS_SKIP=1 LRS_PW_DBG=1" "LRS_SKIP=1 LRS_PW_DBG=2" "LRS_SKIP=1 LRS_PW_DBG=4" "LRS_SKIP=1 LRS_PW_DBG=3" "LRS_SKIP=1 LRS_PW_DBG=6" "LRS_SKIP=1 LRS_PW_DBG=7" "LRS_SKIP=4" > $O/ablate_c4.log 2>&1
  grep -v "^\[lrs\]" $O/ablate_c4.log
}

call_j() {
  mkdir -p gpurun_out/r02j; O=gpurun_out/r02j
  LRS_EXPERIMENTS=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1 || exit 1
  timeout 300 python tools/ablate.py c4 "LRS_SKIP=1" "LRS_SKIP=1 LRS_PW_DBG=5" "LRS_SKIP=1 LRS_PW_DBG=5 LRS_PW_MPC=2 LRS_PW_BP=112" "LRS_SKIP=1 LRS_PW_DBG=7 LRS_PW_MPC=2 LRS_PW_BP=112" > $O/ablate_c4.log 2>&1
  LRS_SKIP=1 LRS_PW_DBG=5 timeout 120 python tools/ptrace.py c4 > $O/ptrace_dbg5.log 2>&1
  LRS_SKIP=1 LRS_PW_DBG=7 timeout 120 python tools/ptrace.py c4 > $O/ptrace_dbg7.log 2>&1
  grep -v "^\[lrs\]" $O/ablate_c4.log
}

call_k() {
  mkdir -p gpurun_out/r02k; O=gpurun_out/r02k
  timeout 300 python -m pytest tests/test_gpu_pw.py -x -q > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
  timeout 300 python tools/ablate.py c4 base "LRS_PW_MPC=2 LRS_PW_BP=112" "LRS_PW_MPC=2 LRS_PW_BP=96" "LRS_PW_MPC=1 LRS_PW_BP=96" > $O/ablate_c4.log 2>&1
  LRS_WCONV_DEBUG=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1
  timeout 120 python tools/ptrace.py c4 > $O/ptrace.log 2>&1
  cat $O/rc.txt; grep -v "^\[lrs\]" $O/ablate_c4.log
}

call_l() {
  mkdir -p gpurun_out/r02l; O=gpurun_out/r02l
  timeout 300 python -m pytest tests/test_gpu_pw.py -x -q > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
  timeout 300 python tools/ablate.py c4 base "LRS_PW_MPC=2 LRS_PW_BP=96" "LRS_PW_MPC=1 LRS_PW_BP=96" "LRS_PW_MPC=2 LRS_PW_BP=64" > $O/ablate_c4.log 2>&1
  LRS_WCONV_DEBUG=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1
  timeout 120 python tools/ptrace.py c4 > $O/ptrace.log 2>&1
  cat $O/rc.txt; grep -v "^\[lrs\]" $O/ablate_c4.log
}

call_m() {
  mkdir -p gpurun_out/r02m; O=gpurun_out/r02m
  LRS_EXPERIMENTS=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1 || exit 1
  timeout 300 python tools/ablate.py c4 "LRS_SKIP=1" "LRS_SKIP=1 LRS_PW_DBG=1" "LRS_SKIP=1 LRS_PW_DBG=2" "LRS_SKIP=1 LRS_PW_DBG=4" "LRS_SKIP=1 LRS_PW_DBG=5" "LRS_SKIP=1 LRS_PW_DBG=6" "LRS_SKIP=1 LRS_PW_DBG=7" "LRS_SKIP=1 LRS_PW_DBG=3" > $O/ablate_c4.log 2>&1
  grep -v "^\[lrs\]" $O/ablate_c4.log
}

call_n() {
  mkdir -p gpurun_out/r02n; O=gpurun_out/r02n
  LRS_EXPERIMENTS=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1 || exit 1
  LRS_SKIP=1 LRS_PW_DBG=7 timeout 120 python tools/ptrace.py c4 > $O/ptrace_dbg7.log 2>&1
  LRS_SKIP=1 LRS_PW_DBG=6 timeout 120 python tools/ptrace.py c4 > $O/ptrace_dbg6.log 2>&1
  LRS_SKIP=1 timeout 120 python tools/ptrace.py c4 > $O/ptrace_dbg0.log 2>&1
}

call_o() {
  mkdir -p gpurun_out/r02o; O=gpurun_out/r02o
  timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "gpu rc=$?" > $O/rc.txt
  timeout 300 python tools/ablate.py c3 base > $O/ablate_c3.log 2>&1
  timeout 300 python tools/ablate.py c2_bf16 base > $O/ablate_c2.log 2>&1
  timeout 300 python tools/ablate.py c4 base "LRS_NO_PW=1" > $O/ablate_c4.log 2>&1
  cat $O/rc.txt; tail -2 $O/pytest_gpu.log; grep -h -v "^\[lrs\]" $O/ablate_*.log
}

call_p() {
  mkdir -p gpurun_out/r02p; O=gpurun_out/r02p
  LRS_WCONV_DEBUG=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1
  timeout 120 python tools/wtrace.py c3 > $O/wtrace_c3.log 2>&1
  LRS_EXPERIMENTS=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build2.log 2>&1
  timeout 300 python tools/ablate.py c3 "LRS_SKIP=1" "LRS_SKIP=1 LRS_WCONV_DBG=1" "LRS_SKIP=1 LRS_WCONV_DBG=66" "LRS_SKIP=1 LRS_WCONV_DBG=67" "LRS_SKIP=1 LRS_WCONV_DBG=8" > $O/ablate_c3.log 2>&1
  grep -v "^\[lrs\]" $O/ablate_c3.log
}

call_p1() {
  mkdir -p gpurun_out/r02p1; O=gpurun_out/r02p1
  timeout 60 ./tools/probe_2cta 0 > $O/mode0.log 2>&1; echo "rc0=$?" >> $O/mode0.log
  timeout 60 ./tools/probe_2cta 1 > $O/mode1.log 2>&1; echo "rc1=$?" >> $O/mode1.log
  cat $O/mode0.log $O/mode1.log
}

call_p2() {
  mkdir -p gpurun_out/r02p2; O=gpurun_out/r02p2
  timeout 120 ./tools/probe_2cta_rate > $O/rate.log 2>&1; echo "rc=$?" >> $O/rate.log
  cat $O/rate.log
}

call_p3() {
  mkdir -p gpurun_out/r02p3; O=gpurun_out/r02p3
  LRS_VERBOSE=1 timeout 120 python -m pytest tests/test_gpu_sparse_tc.py -x -q -k "pair" > $O/pytest_pair.log 2>&1; echo "pair rc=$?" > $O/rc.txt
  cat $O/rc.txt; tail -30 $O/pytest_pair.log | grep -v "^\[lrs\]" | tail -25
}

call_p4() {
  mkdir -p gpurun_out/r02p4; O=gpurun_out/r02p4
  timeout 120 python -m pytest tests/test_gpu_sparse_tc.py -x -q -k "pair" > $O/pytest_pair.log 2>&1; echo "pair rc=$?" > $O/rc.txt
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_PAIR=0" "LRS_WCONV_PAIR=1" > $O/ablate_c3.log 2>&1
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_bf16 base "LRS_WCONV_PAIR=0" "LRS_WCONV_PAIR=1" > $O/ablate_c2.log 2>&1
  cat $O/rc.txt; tail -3 $O/pytest_pair.log; grep "wconv plan\|c3 \[\|c2_bf16 \[" $O/ablate_c3.log $O/ablate_c2.log
}

call_p5() {
  mkdir -p gpurun_out/r02p5; O=gpurun_out/r02p5
  LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
  LRS_WCONV_PAIR=1 timeout 300 python tools/wtrace.py c3 > $O/wtrace_pair.log 2>&1
  LRS_WCONV_PAIR=1 LRS_NO_EARLY=1 timeout 300 python tools/wtrace.py c3 > $O/wtrace_pair_noearly.log 2>&1
  cut -c1-900 $O/wtrace_pair.log | head -8; head -2 $O/wtrace_pair_noearly.log
}

call_p6() {
  mkdir -p gpurun_out/r02p6; O=gpurun_out/r02p6
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 "LRS_WCONV_PAIR=1 LRS_WCONV_BPI=2" "LRS_WCONV_PAIR=1 LRS_WCONV_BPI=2 LRS_WCONV_NS=3" "LRS_WCONV_PAIR=1 LRS_WCONV_NWB1=1" "LRS_WCONV_PAIR=1 LRS_WCONV_BPI=2 LRS_WCONV_NWB1=1" > $O/ablate_c3.log 2>&1
  grep "wconv plan\|c3 \[" $O/ablate_c3.log
}

call_p7() {
  mkdir -p gpurun_out/r02p7; O=gpurun_out/r02p7
  timeout 120 ./tools/probe_2cta_rate > $O/rate.log 2>&1; echo "rc=$?" >> $O/rate.log
  cat $O/rate.log
}

call_p8() {
  mkdir -p gpurun_out/r02p8; O=gpurun_out/r02p8
  LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
  LRS_WCONV_PAIR=1 timeout 300 python tools/wtrace.py c3 > $O/wtrace_pair.log 2>&1
  timeout 300 python tools/wtrace.py c3 > $O/wtrace_single.log 2>&1
  grep "mma items" $O/wtrace_pair.log | cut -c1-1500; grep "mma items" $O/wtrace_single.log | cut -c1-1500
}

call_p9() {
  mkdir -p gpurun_out/r02p9; O=gpurun_out/r02p9
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "gpu rc=$?" > $O/rc.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
  cat $O/rc.txt; tail -3 $O/pytest_gpu.log; tail -8 $O/smoke.log
}

call_q() {
  mkdir -p gpurun_out/r02q; O=gpurun_out/r02q
  timeout 300 python -m pytest tests/test_gpu_bounds.py -q > $O/pytest_bounds.log 2>&1; echo "bounds rc=$?" > $O/rc.txt
  timeout 2400 python tools/f2_speed_bound.py > $O/f2.log 2>&1; echo "f2 rc=$?" >> $O/rc.txt
  cp profiles/r02_f2_speed_bound.json $O/ 2>/dev/null
  cat $O/rc.txt; tail -3 $O/pytest_bounds.log; tail -12 $O/f2.log
}

call_q1() {
  mkdir -p gpurun_out/r02q1; O=gpurun_out/r02q1
  timeout 300 python tools/ablate.py c3 base "LRS_CORE_GRID=43" "LRS_CORE_GRID=64" "LRS_CORE_GRID=96" "LRS_CORE_GRID=128" "LRS_CORE_GRID=43 LRS_CORE_IPT=2 LRS_CORE_TH=7" "LRS_CORE_GRID=64 LRS_CORE_IPT=2 LRS_CORE_TH=7" > $O/ablate_c3.log 2>&1
  timeout 300 python tools/ablate.py c2_bf16 base "LRS_CORE_GRID=24" "LRS_CORE_GRID=48" "LRS_CORE_GRID=64" > $O/ablate_c2.log 2>&1
  grep "\[" $O/ablate_c3.log $O/ablate_c2.log
}

call_q2() {
  mkdir -p gpurun_out/r02q2; O=gpurun_out/r02q2
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 "LRS_WCONV_PAIR=1 LRS_WCONV_BPI=2 LRS_WCONV_NS=2" "LRS_WCONV_PAIR=1 LRS_WCONV_BPI=1 LRS_WCONV_NS=3" > $O/ablate_c3.log 2>&1
  grep "wconv plan\|c3 \[" $O/ablate_c3.log
}

call_r() {
  mkdir -p gpurun_out/r02r; O=gpurun_out/r02r
  timeout 300 python -m pytest tests/test_gpu_pw.py tests/test_gpu_bounds.py -q -x > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_TH=4" "LRS_WCONV_TH=5" "LRS_WCONV_TH=3" > $O/ablate_c3.log 2>&1
  timeout 2400 python tools/f2_speed_bound.py > $O/f2.log 2>&1; echo "f2 rc=$?" >> $O/rc.txt
  cp profiles/r02_f2_speed_bound.json $O/ 2>/dev/null
  cat $O/rc.txt; tail -3 $O/pytest_pw.log; grep "c3 \[\|wconv plan" $O/ablate_c3.log; tail -12 $O/f2.log
}

call_s() {
  mkdir -p gpurun_out/r02s; O=gpurun_out/r02s
  timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "gpu rc=$?" > $O/rc.txt
  for c in c3 c2_bf16 c4; do
    timeout 600 python bench.py --config $c --steps 200 --warmup 10 --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?" >> $O/rc.txt
  done
  timeout 2400 python tools/f2_speed_bound.py > $O/f2.log 2>&1; echo "f2 rc=$?" >> $O/rc.txt
  cp profiles/r02_f2_speed_bound.json $O/ 2>/dev/null
  cat $O/rc.txt; tail -2 $O/pytest_gpu.log; tail -12 $O/f2.log
}

call_san1() {
  mkdir -p gpurun_out/r02san; O=gpurun_out/r02san
  export LRS_NO_AUTOTUNE=1
  timeout 300 python tools/sanitize_run.py > $O/plain.log 2>&1 && \
  timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_run.py > $O/racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/rc.txt
  tail -5 $O/racecheck.log
}

call_t() {
  mkdir -p gpurun_out/r02t; O=gpurun_out/r02t
  timeout 300 python -m pytest tests/test_gpu_sparse_tc.py -q -x > $O/pytest_tc.log 2>&1; echo "tc rc=$?" > $O/rc.txt
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_IPW=8" "LRS_WCONV_IPW=4" > $O/ablate_c3.log 2>&1
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_bf16 "LRS_WCONV_IPW=8" "LRS_WCONV_IPW=4" > $O/ablate_c2.log 2>&1
  cat $O/rc.txt; tail -3 $O/pytest_tc.log; grep -h "\] \|wconv plan" $O/ablate_c3.log $O/ablate_c2.log | grep -v "\[lrs\] core\|autotune"
}

call_u() {
  mkdir -p gpurun_out/r02u; O=gpurun_out/r02u
  LRS_VERBOSE=1 timeout 600 python tools/ablate.py c3 "LRS_WCONV_IPW=8 LRS_WCONV_TH=7" "LRS_WCONV_IPW=4 LRS_WCONV_BPI=2" "LRS_WCONV_IPW=4 LRS_WCONV_BPI=2 LRS_WCONV_NS=4" "LRS_WCONV_IPW=4 LRS_WCONV_TH=4" "LRS_WCONV_IPW=4 LRS_WCONV_BPI=2 LRS_WCONV_TH=4" > $O/ablate_c3.log 2>&1
  LRS_VERBOSE=1 timeout 600 python tools/ablate.py c2_bf16 "LRS_WCONV_IPW=8 LRS_WCONV_TH=7" "LRS_WCONV_IPW=8 LRS_WCONV_TH=4" "LRS_WCONV_IPW=4 LRS_WCONV_BPI=2" "LRS_WCONV_IPW=4 LRS_WCONV_TH=7" "LRS_WCONV_IPW=4 LRS_WCONV_TH=4 LRS_WCONV_BPI=2" > $O/ablate_c2.log 2>&1
  LRS_VERBOSE=1 timeout 600 python tools/ablate.py c4 "LRS_NO_PW=1 LRS_WCONV_IPW=8" "LRS_NO_PW=1 LRS_WCONV_IPW=4" > $O/ablate_c4.log 2>&1
  grep -h "\] \|wconv plan" $O/ablate_c3.log $O/ablate_c2.log $O/ablate_c4.log | grep -v "\[lrs\] core\|autotune"
}

call_w() {
  mkdir -p gpurun_out/r02w; O=gpurun_out/r02w
  LRS_VERBOSE=1 timeout 300 python -m pytest tests/test_gpu_pw.py -x -q > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
  timeout 300 python tools/ablate.py c4 base "LRS_PW_FT=0" > $O/ablate_c4.log 2>&1
  cat $O/rc.txt; tail -15 $O/pytest_pw.log | grep -v "^\[lrs\] \(core\|tiny\|spadd\|autotune\)"; grep "c4 \[" $O/ablate_c4.log
}

call_x() {
  mkdir -p gpurun_out/r02x; O=gpurun_out/r02x
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_parity.log 2>&1; echo "parity rc=$?" > $O/rc.txt
  timeout 2400 python tools/f2_speed_bound.py > $O/f2.log 2>&1; echo "f2 rc=$?" >> $O/rc.txt
  cp profiles/r02_f2_speed_bound.json $O/ 2>/dev/null
  cat $O/rc.txt; tail -3 $O/pytest_parity.log; grep "^x3 L [1-9]\|^x3 L1[01]" $O/f2.log | head -12; tail -12 $O/f2.log
}

call_y() {
  mkdir -p gpurun_out/r02y; O=gpurun_out/r02y
  timeout 300 python -m pytest tests/test_gpu_pw.py tests/test_gpu_bounds.py -x -q > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c4 base "LRS_PW_EPIBUF=2" "LRS_PW_EPIBUF=1" "LRS_PW_MPC=2 LRS_PW_BP=96" "LRS_PW_MPC=1 LRS_PW_BP=96" > $O/ablate_c4.log 2>&1
  cat $O/rc.txt; tail -2 $O/pytest_pw.log; grep "pw plan\|c4 \[" $O/ablate_c4.log
}

call_z() {
  mkdir -p gpurun_out/r02z; O=gpurun_out/r02z
  timeout 600 python -m pytest tests/test_gpu_spadd_f32.py tests/test_gpu_parity.py tests/test_gpu_bounds.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  timeout 300 python tools/ablate.py c2_f32 base > $O/ablate.log 2>&1
  cat $O/rc.txt; tail -2 $O/pytest.log; grep "c2_f32 \[" $O/ablate.log
}

call_q3() {
  mkdir -p gpurun_out/r02q3; O=gpurun_out/r02q3
  LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
  E="LRS_SKIP=1 LRS_PW_MPC=2 LRS_PW_BP=96 LRS_PW_CPI=2"
  timeout 300 python tools/ablate.py c4 "$E" "$E LRS_PW_DBG=1" "$E LRS_PW_DBG=9" "$E LRS_PW_DBG=25" "$E LRS_PW_DBG=57" "$E LRS_PW_DBG=7" "$E LRS_PW_DBG=63" "$E LRS_PW_DBG=6" > $O/ablate.log 2>&1
  grep "c4 \[" $O/ablate.log
}

call_q4() {
  mkdir -p gpurun_out/r02q4; O=gpurun_out/r02q4
  timeout 900 python -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_bench_pattern.py tests/test_gpu_overlap.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  timeout 300 python tools/ablate.py c3 base base > $O/ablate_c3.log 2>&1
  cat $O/rc.txt; tail -2 $O/pytest.log; grep "c3 \[" $O/ablate_c3.log
}

call_q5() {
  mkdir -p gpurun_out/r02q5; O=gpurun_out/r02q5
  timeout 600 python -m pytest $(grep -ln "forward_host" tests/test_gpu*.py) -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-dense > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench rc=$?" >> $O/rc.txt
  timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu --no-dense > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?" >> $O/rc.txt
  cat $O/rc.txt; tail -2 $O/pytest.log; python -c "
  import json
  for c in ('c3','c4'):
      d=json.loads(open('$O/bench_'+c+'.json').read().strip().splitlines()[-1]); print(c, round(d['value']), 'e2e', round(d['e2e']['value']), d['verify'].get('e2e_bitwise_device_forward'))"
}

call_q6() {
  mkdir -p gpurun_out/r02q6; O=gpurun_out/r02q6
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_TH=4" "LRS_WCONV_TH=3" "LRS_WCONV_TH=4 LRS_WCONV_IPW=4" > $O/ablate_c3.log 2>&1
  grep "wconv plan\|c3 \[" $O/ablate_c3.log
}

call_q7() {
  mkdir -p gpurun_out/r02q7; O=gpurun_out/r02q7
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 "CFG_batch=32" "CFG_batch=32 LRS_WCONV_IPW=4" "CFG_batch=32 LRS_WCONV_TH=4" "CFG_batch=32 LRS_WCONV_IPW=4 LRS_WCONV_TH=4" "CFG_batch=64" "CFG_batch=128" > $O/ablate_c3.log 2>&1
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_bf16 "CFG_batch=8" "CFG_batch=16" "CFG_batch=32" > $O/ablate_c2.log 2>&1
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c4 "CFG_batch=16" "CFG_batch=32" "CFG_batch=64" > $O/ablate_c4.log 2>&1
  grep "wconv plan\|pw plan\|\]" $O/ablate_c3.log $O/ablate_c2.log $O/ablate_c4.log | grep -v autotune
}

call_q8() {
  mkdir -p gpurun_out/r02q8; O=gpurun_out/r02q8
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_TH=2" "LRS_WCONV_TH=1" "CFG_batch=128 LRS_WCONV_TH=7" > $O/ablate_c3.log 2>&1
  grep "wconv plan\|c3 \[" $O/ablate_c3.log
}

call_q9() {
  mkdir -p gpurun_out/r02q9; O=gpurun_out/r02q9
  timeout 900 python -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_bench_pattern.py tests/test_gpu_overlap.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "CFG_batch=128" "CFG_batch=64" "CFG_batch=32" > $O/ablate_c3.log 2>&1
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_bf16 base "CFG_batch=32" "CFG_batch=16" "CFG_batch=8" > $O/ablate_c2.log 2>&1
  cat $O/rc.txt; tail -2 $O/pytest.log; grep "autotune wconv\|c3 \[\|c2_bf16 \[" $O/ablate_c3.log $O/ablate_c2.log
}

call_r1() {
  mkdir -p gpurun_out/r02r1; O=gpurun_out/r02r1
  LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_CORE_IPT=1 LRS_CORE_TH=7" "LRS_CORE_IPT=2 LRS_CORE_TH=7" "LRS_CORE_IPT=1 LRS_CORE_TH=4" "LRS_CORE_IPT=1 LRS_CORE_TH=7 LRS_CORE_GRID=148" > $O/ablate_c3.log 2>&1
  grep "core:\|c3 \[" $O/ablate_c3.log | grep -v autotune | tail -12
}

call_r2() {
  mkdir -p gpurun_out/r02r2; O=gpurun_out/r02r2
  timeout 300 python tools/ablate.py c3 base base > $O/ablate_c3.log 2>&1
  timeout 300 python tools/ablate.py c2_bf16 base base > $O/ablate_c2.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_bench_pattern.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  cat $O/rc.txt; tail -2 $O/pytest.log; grep "\[" $O/ablate_c3.log $O/ablate_c2.log
}

call_s1() {
  mkdir -p gpurun_out/r02s1; O=gpurun_out/r02s1
  LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
  timeout 300 python tools/ctrace.py c3 > $O/ctrace_c3.log 2>&1
  cat $O/ctrace_c3.log
}

call_s2() {
  mkdir -p gpurun_out/r02s2; O=gpurun_out/r02s2
  timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" > $O/rc.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
  timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?" >> $O/rc.txt
  cat $O/rc.txt; tail -1 $O/pytest_gpu.log
}

call_t1() {
  mkdir -p gpurun_out/r02t1; O=gpurun_out/r02t1
  timeout 600 python -m pytest tests/test_gpu_sparse_tc.py -x -q -k "tma_store" > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  timeout 300 python tools/ablate.py c3 base "LRS_WCONV_EPI_TMA=1" > $O/ablate_c3.log 2>&1
  timeout 300 python tools/ablate.py c2_bf16 base "LRS_WCONV_EPI_TMA=1" > $O/ablate_c2.log 2>&1
  cat $O/rc.txt; tail -3 $O/pytest.log; grep "\[" $O/ablate_c3.log $O/ablate_c2.log
}

call_u1() {
  mkdir -p gpurun_out/r02u1; O=gpurun_out/r02u1
  timeout 300 python tools/ablate.py c3 base base > $O/ablate_c3.log 2>&1
  timeout 300 python tools/ablate.py c2_bf16 base base > $O/ablate_c2.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_parity.py tests/test_gpu_bench_pattern.py tests/test_gpu_overlap.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  cat $O/rc.txt; tail -2 $O/pytest.log; grep "\[" $O/ablate_c3.log $O/ablate_c2.log
}

call_u2() {
  mkdir -p gpurun_out/r02u2; O=gpurun_out/r02u2
  timeout 300 python tools/ablate.py c3 base "LRS_WCONV_DENSE_LAST=1" base > $O/ablate_c3.log 2>&1
  timeout 300 python tools/ablate.py c2_bf16 base "LRS_WCONV_DENSE_LAST=1" > $O/ablate_c2.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_parity.py tests/test_gpu_bench_pattern.py tests/test_gpu_overlap.py tests/test_gpu_pw.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  cat $O/rc.txt; tail -2 $O/pytest.log; grep "\[" $O/ablate_c3.log $O/ablate_c2.log
}

call_v1() {
  mkdir -p gpurun_out/r02v1; O=gpurun_out/r02v1
  timeout 900 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_pw.py tests/test_gpu_bench_pattern.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  timeout 300 python tools/ablate.py c4 base "LRS_NO_EARLY=1" base > $O/ablate_c4.log 2>&1
  cat $O/rc.txt; tail -3 $O/pytest.log; grep "c4 \[" $O/ablate_c4.log
}

call_v2() {
  mkdir -p gpurun_out/r02v2; O=gpurun_out/r02v2
  timeout 600 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_parity.py tests/test_gpu_cp.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  timeout 300 python tools/ablate.py c1 base "LRS_NO_EARLY=1" base > $O/ablate_c1.log 2>&1
  cat $O/rc.txt; tail -3 $O/pytest.log; grep "c1 \[" $O/ablate_c1.log
}

call_v3() {
  mkdir -p gpurun_out/r02v3; O=gpurun_out/r02v3
  LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
  timeout 300 python tools/wtrace.py c2_bf16 > $O/wtrace_c2.log 2>&1
  timeout 300 python tools/ctrace.py c2_bf16 > $O/ctrace_c2.log 2>&1
  grep -v "^\[lrs\]\|plan" $O/wtrace_c2.log | cut -c1-600 | head -5; cat $O/ctrace_c2.log
}

call_v4() {
  mkdir -p gpurun_out/r02v4; O=gpurun_out/r02v4
  timeout 300 python tools/ablate.py c3 base base > $O/ablate_c3.log 2>&1
  timeout 300 python tools/ablate.py c2_bf16 base base > $O/ablate_c2.log 2>&1
  timeout 900 python -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_parity.py tests/test_gpu_bench_pattern.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
  cat $O/rc.txt; tail -2 $O/pytest.log; grep "\[" $O/ablate_c3.log $O/ablate_c2.log
}

