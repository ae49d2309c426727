mkdir -p gpurun_out/r02q4; O=gpurun_out/r02q4
timeout 900 python -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_bench_pattern.py tests/test_gpu_overlap.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
timeout 300 python tools/ablate.py c3 base base > $O/ablate_c3.log 2>&1
cat $O/rc.txt; tail -2 $O/pytest.log; grep "c3 \[" $O/ablate_c3.log
