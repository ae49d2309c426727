mkdir -p gpurun_out/r02n; O=gpurun_out/r02n
LRS_EXPERIMENTS=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1 || exit 1
LRS_SKIP=1 LRS_PW_DBG=7 timeout 120 python tools/ptrace.py c4 > $O/ptrace_dbg7.log 2>&1
LRS_SKIP=1 LRS_PW_DBG=6 timeout 120 python tools/ptrace.py c4 > $O/ptrace_dbg6.log 2>&1
LRS_SKIP=1 timeout 120 python tools/ptrace.py c4 > $O/ptrace_dbg0.log 2>&1
