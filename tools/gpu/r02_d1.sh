mkdir -p gpurun_out/r02d1; O=gpurun_out/r02d1
timeout 600 python -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_parity.py tests/test_gpu_bench_pattern.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_EPI=scratch" "LRS_WCONV_EPI=direct" "LRS_WCONV_EPI=direct LRS_WCONV_NS=3" > $O/ablate_c3.log 2>&1
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_bf16 base "LRS_WCONV_EPI=scratch" "LRS_WCONV_EPI=direct" > $O/ablate_c2.log 2>&1
cat $O/rc.txt; tail -3 $O/pytest.log; grep "wconv plan\|c3 \[\|c2_bf16 \[" $O/ablate_c3.log $O/ablate_c2.log
