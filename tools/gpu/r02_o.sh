mkdir -p gpurun_out/r02o; O=gpurun_out/r02o
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "gpu rc=$?" > $O/rc.txt
timeout 300 python tools/ablate.py c3 base > $O/ablate_c3.log 2>&1
timeout 300 python tools/ablate.py c2_bf16 base > $O/ablate_c2.log 2>&1
timeout 300 python tools/ablate.py c4 base "LRS_NO_PW=1" > $O/ablate_c4.log 2>&1
cat $O/rc.txt; tail -2 $O/pytest_gpu.log; grep -h -v "^\[lrs\]" $O/ablate_*.log
