mkdir -p gpurun_out/r02t; O=gpurun_out/r02t
timeout 300 python -m pytest tests/test_gpu_sparse_tc.py -q -x > $O/pytest_tc.log 2>&1; echo "tc rc=$?" > $O/rc.txt
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_IPW=8" "LRS_WCONV_IPW=4" > $O/ablate_c3.log 2>&1
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_bf16 "LRS_WCONV_IPW=8" "LRS_WCONV_IPW=4" > $O/ablate_c2.log 2>&1
cat $O/rc.txt; tail -3 $O/pytest_tc.log; grep -h "\] \|wconv plan" $O/ablate_c3.log $O/ablate_c2.log | grep -v "\[lrs\] core\|autotune"
