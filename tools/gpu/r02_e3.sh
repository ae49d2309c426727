mkdir -p gpurun_out/r02e3; O=gpurun_out/r02e3
timeout 900 python -m pytest tests/test_gpu_core_fused.py tests/test_gpu_parity.py tests/test_gpu_bench_pattern.py tests/test_gpu_overlap.py tests/test_gpu_cp.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_CORE_SPLIT_RING=1" > $O/ablate_c3.log 2>&1
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c2_bf16 base "LRS_CORE_SPLIT_RING=1" > $O/ablate_c2.log 2>&1
cat $O/rc.txt; tail -3 $O/pytest.log; grep "c3 \[\|c2_bf16 \[" $O/ablate_c3.log $O/ablate_c2.log; grep "core:" $O/ablate_c3.log | sort | uniq -c | head
