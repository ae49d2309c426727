mkdir -p gpurun_out/r02g1; O=gpurun_out/r02g1
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_GATHER=0" "LRS_WCONV_GATHER=1" > $O/ablate_c3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_pw.py tests/test_gpu_parity.py tests/test_gpu_bench_pattern.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
cat $O/rc.txt; tail -15 $O/pytest.log; grep "wconv plan\|c3 \[\|rror" $O/ablate_c3.log
