# round 2, call F: pw timeline (debug build) + pw tests
mkdir -p gpurun_out/r02f; O=gpurun_out/r02f
timeout 300 python -m pytest tests/test_gpu_pw.py -x -q > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
LRS_WCONV_DEBUG=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1
LRS_VERBOSE=1 timeout 120 python tools/ptrace.py c4 > $O/ptrace_c4.log 2>&1
LRS_PW_MPC=2 LRS_PW_BP=112 timeout 120 python tools/ptrace.py c4 > $O/ptrace_c4_m2.log 2>&1
cat $O/rc.txt
