mkdir -p gpurun_out/r02p5; O=gpurun_out/r02p5
LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
LRS_WCONV_PAIR=1 timeout 300 python tools/wtrace.py c3 > $O/wtrace_pair.log 2>&1
LRS_WCONV_PAIR=1 LRS_NO_EARLY=1 timeout 300 python tools/wtrace.py c3 > $O/wtrace_pair_noearly.log 2>&1
cut -c1-900 $O/wtrace_pair.log | head -8; head -2 $O/wtrace_pair_noearly.log
