mkdir -p gpurun_out/r02j; O=gpurun_out/r02j
LRS_EXPERIMENTS=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1 || exit 1
timeout 300 python tools/ablate.py c4 "LRS_SKIP=1" "LRS_SKIP=1 LRS_PW_DBG=5" "LRS_SKIP=1 LRS_PW_DBG=5 LRS_PW_MPC=2 LRS_PW_BP=112" "LRS_SKIP=1 LRS_PW_DBG=7 LRS_PW_MPC=2 LRS_PW_BP=112" > $O/ablate_c4.log 2>&1
LRS_SKIP=1 LRS_PW_DBG=5 timeout 120 python tools/ptrace.py c4 > $O/ptrace_dbg5.log 2>&1
LRS_SKIP=1 LRS_PW_DBG=7 timeout 120 python tools/ptrace.py c4 > $O/ptrace_dbg7.log 2>&1
grep -v "^\[lrs\]" $O/ablate_c4.log
