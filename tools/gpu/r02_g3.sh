mkdir -p gpurun_out/r02g3; O=gpurun_out/r02g3
LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
timeout 300 python tools/wtrace.py c3 > $O/wtrace_c3.log 2>&1
LRS_WCONV_GATHER=0 timeout 300 python tools/wtrace.py c3 > $O/wtrace_c3_res.log 2>&1
LRS_NO_AUTOTUNE=1 timeout 300 python tools/wtrace.py c3 > $O/wtrace_c3_noat.log 2>&1
cat $O/wtrace_c3.log | head -4; head -2 $O/wtrace_c3_res.log;  head -2 $O/wtrace_c3_noat.log
