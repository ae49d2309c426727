mkdir -p gpurun_out/r02p8; O=gpurun_out/r02p8
LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
LRS_WCONV_PAIR=1 timeout 300 python tools/wtrace.py c3 > $O/wtrace_pair.log 2>&1
timeout 300 python tools/wtrace.py c3 > $O/wtrace_single.log 2>&1
grep "mma items" $O/wtrace_pair.log | cut -c1-1500; grep "mma items" $O/wtrace_single.log | cut -c1-1500
