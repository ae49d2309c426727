mkdir -p gpurun_out/r02e1; O=gpurun_out/r02e1
timeout 600 python -m pytest tests/test_gpu_overlap.py -x -q > $O/pytest_overlap.log 2>&1; echo "overlap rc=$?" > $O/rc.txt
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_NO_EARLY=1" > $O/ablate_c3.log 2>&1
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_bf16 base "LRS_NO_EARLY=1" > $O/ablate_c2.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "gpu rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -3 $O/pytest_overlap.log; tail -3 $O/pytest_gpu.log; grep "autotune\|c3 \[\|c2_bf16 \[" $O/ablate_c3.log $O/ablate_c2.log
