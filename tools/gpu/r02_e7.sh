mkdir -p gpurun_out/r02e7; O=gpurun_out/r02e7
LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
LRS_PW_MPC=2 LRS_PW_BP=96 LRS_PW_CPI=2 timeout 300 python tools/ptrace.py c4 > $O/ptrace_a.log 2>&1
LRS_PW_MPC=2 LRS_PW_BP=96 LRS_PW_CPI=2 LRS_PW_DBG=7 timeout 300 python tools/ptrace.py c4 > $O/ptrace_dbg7.log 2>&1
LRS_PW_MPC=2 LRS_PW_BP=96 LRS_PW_CPI=2 timeout 300 python tools/ablate.py c4 base "LRS_SKIP=1" "LRS_SKIP=1 LRS_PW_DBG=1" "LRS_SKIP=1 LRS_PW_DBG=2" "LRS_SKIP=1 LRS_PW_DBG=4" "LRS_SKIP=1 LRS_PW_DBG=7" > $O/ablate.log 2>&1
cat $O/ptrace_a.log $O/ptrace_dbg7.log | cut -c1-600; grep "c4 \[" $O/ablate.log
