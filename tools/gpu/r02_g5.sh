mkdir -p gpurun_out/r02g5; O=gpurun_out/r02g5
LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
timeout 300 python tools/ctrace.py c3 > $O/ctrace_c3.log 2>&1
LRS_CORE_IPT=1 LRS_CORE_TH=7 timeout 300 python tools/ctrace.py c3 > $O/ctrace_c3_ipt1.log 2>&1
LRS_CORE_IPT=2 LRS_CORE_TH=7 timeout 300 python tools/ctrace.py c3 > $O/ctrace_c3_ipt2.log 2>&1
cat $O/ctrace_c3*.log
