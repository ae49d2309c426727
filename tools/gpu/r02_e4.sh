mkdir -p gpurun_out/r02e4; O=gpurun_out/r02e4
timeout 300 python tools/ablate.py c4 base > $O/ablate_c4.log 2>&1
timeout 300 python tools/ablate.py c3 base > $O/ablate_c3.log 2>&1
timeout 300 python tools/ablate.py c2_bf16 base > $O/ablate_c2.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "gpu rc=$?" > $O/rc.txt
cat $O/rc.txt; tail -3 $O/pytest_gpu.log; grep "\[" $O/ablate_c4.log $O/ablate_c3.log $O/ablate_c2.log
