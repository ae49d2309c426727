mkdir -p gpurun_out/r02w; O=gpurun_out/r02w
LRS_VERBOSE=1 timeout 300 python -m pytest tests/test_gpu_pw.py -x -q > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
timeout 300 python tools/ablate.py c4 base "LRS_PW_FT=0" > $O/ablate_c4.log 2>&1
cat $O/rc.txt; tail -15 $O/pytest_pw.log | grep -v "^\[lrs\] \(core\|tiny\|spadd\|autotune\)"; grep "c4 \[" $O/ablate_c4.log
