mkdir -p gpurun_out/r02f3; O=gpurun_out/r02f3
LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
LRS_VERBOSE=1 timeout 300 python tools/wtrace.py c2_bf16 > $O/wtrace_c2.log 2>&1
timeout 300 python tools/ctrace.py c2_bf16 > $O/ctrace_c2.log 2>&1
grep "plan\|core:" $O/wtrace_c2.log | tail -3; grep -v "^\[lrs\]\|plan" $O/wtrace_c2.log | cut -c1-700 | head -8; cat $O/ctrace_c2.log
