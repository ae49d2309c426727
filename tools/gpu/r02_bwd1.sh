mkdir -p gpurun_out/bwd1; O=gpurun_out/bwd1
LRS_VERBOSE=1 timeout 900 python -m pytest tests/test_gpu_backward.py -x -q -k "small_3x3 and matches" > $O/t1.log 2>&1; echo "t1 rc=$?" >> $O/rc.txt
timeout 1200 python -m pytest tests/test_gpu_backward.py -q > $O/all.log 2>&1; echo "all rc=$?" >> $O/rc.txt
cat $O/rc.txt
