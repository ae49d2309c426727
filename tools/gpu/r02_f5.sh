mkdir -p gpurun_out/r02f5; O=gpurun_out/r02f5
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c4 base "LRS_A1_MB1=1" > $O/ablate_c4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pw.py tests/test_gpu_bench_pattern.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
cat $O/rc.txt; tail -3 $O/pytest.log; grep "c4 \[" $O/ablate_c4.log
