mkdir -p gpurun_out/r02r; O=gpurun_out/r02r
timeout 300 python -m pytest tests/test_gpu_pw.py tests/test_gpu_bounds.py -q -x > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_TH=4" "LRS_WCONV_TH=5" "LRS_WCONV_TH=3" > $O/ablate_c3.log 2>&1
timeout 2400 python tools/f2_speed_bound.py > $O/f2.log 2>&1; echo "f2 rc=$?" >> $O/rc.txt
cp profiles/r02_f2_speed_bound.json $O/ 2>/dev/null
cat $O/rc.txt; tail -3 $O/pytest_pw.log; grep "c3 \[\|wconv plan" $O/ablate_c3.log; tail -12 $O/f2.log
