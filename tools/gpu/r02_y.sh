mkdir -p gpurun_out/r02y; O=gpurun_out/r02y
timeout 300 python -m pytest tests/test_gpu_pw.py tests/test_gpu_bounds.py -x -q > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c4 base "LRS_PW_EPIBUF=2" "LRS_PW_EPIBUF=1" "LRS_PW_MPC=2 LRS_PW_BP=96" "LRS_PW_MPC=1 LRS_PW_BP=96" > $O/ablate_c4.log 2>&1
cat $O/rc.txt; tail -2 $O/pytest_pw.log; grep "pw plan\|c4 \[" $O/ablate_c4.log
