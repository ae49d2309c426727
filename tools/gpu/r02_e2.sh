mkdir -p gpurun_out/r02e2; O=gpurun_out/r02e2
LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
timeout 300 python tools/wtrace.py c3 > $O/wtrace_c3.log 2>&1
timeout 300 python tools/ctrace.py c3 > $O/ctrace_c3.log 2>&1
cat $O/wtrace_c3.log | head -3; cat $O/ctrace_c3.log
