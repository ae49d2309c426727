mkdir -p gpurun_out/r02p4; O=gpurun_out/r02p4
timeout 120 python -m pytest tests/test_gpu_sparse_tc.py -x -q -k "pair" > $O/pytest_pair.log 2>&1; echo "pair rc=$?" > $O/rc.txt
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_PAIR=0" "LRS_WCONV_PAIR=1" > $O/ablate_c3.log 2>&1
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_bf16 base "LRS_WCONV_PAIR=0" "LRS_WCONV_PAIR=1" > $O/ablate_c2.log 2>&1
cat $O/rc.txt; tail -3 $O/pytest_pair.log; grep "wconv plan\|c3 \[\|c2_bf16 \[" $O/ablate_c3.log $O/ablate_c2.log
