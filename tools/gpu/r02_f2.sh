mkdir -p gpurun_out/r02f2; O=gpurun_out/r02f2
timeout 900 python -m pytest tests/test_gpu_pw.py tests/test_gpu_sparse_tc.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c4 base "LRS_NO_AUTOTUNE=1" "LRS_NO_SPTC=1" > $O/ablate_c4.log 2>&1
timeout 300 python tools/ablate.py c2_bf16 base "LRS_NO_SPTC=1" > $O/ablate_c2.log 2>&1
timeout 300 python tools/ablate.py c3 base "LRS_NO_SPTC=1" > $O/ablate_c3.log 2>&1
cat $O/rc.txt; tail -2 $O/pytest.log; grep "autotune pw\|\[" $O/ablate_c4.log | grep -v "core:" ; grep "\[" $O/ablate_c2.log $O/ablate_c3.log
