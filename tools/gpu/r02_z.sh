mkdir -p gpurun_out/r02z; O=gpurun_out/r02z
timeout 600 python -m pytest tests/test_gpu_spadd_f32.py tests/test_gpu_parity.py tests/test_gpu_bounds.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
timeout 300 python tools/ablate.py c2_f32 base > $O/ablate.log 2>&1
cat $O/rc.txt; tail -2 $O/pytest.log; grep "c2_f32 \[" $O/ablate.log
