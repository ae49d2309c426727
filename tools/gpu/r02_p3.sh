mkdir -p gpurun_out/r02p3; O=gpurun_out/r02p3
LRS_VERBOSE=1 timeout 120 python -m pytest tests/test_gpu_sparse_tc.py -x -q -k "pair" > $O/pytest_pair.log 2>&1; echo "pair rc=$?" > $O/rc.txt
cat $O/rc.txt; tail -30 $O/pytest_pair.log | grep -v "^\[lrs\]" | tail -25
