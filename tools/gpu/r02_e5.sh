mkdir -p gpurun_out/r02e5; O=gpurun_out/r02e5
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c4 base "LRS_PW_CPI=1" "LRS_PW_CPI=2" "LRS_PW_CPI=4" > $O/ablate_c4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pw.py tests/test_gpu_bench_pattern.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
cat $O/rc.txt; tail -3 $O/pytest.log; grep "pw plan\|c4 \[" $O/ablate_c4.log
