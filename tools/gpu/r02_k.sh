mkdir -p gpurun_out/r02k; O=gpurun_out/r02k
timeout 300 python -m pytest tests/test_gpu_pw.py -x -q > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
timeout 300 python tools/ablate.py c4 base "LRS_PW_MPC=2 LRS_PW_BP=112" "LRS_PW_MPC=2 LRS_PW_BP=96" "LRS_PW_MPC=1 LRS_PW_BP=96" > $O/ablate_c4.log 2>&1
LRS_WCONV_DEBUG=1 python -c "from paper_2006_06443_b200 import _build; _build.build(force=True)" > $O/build.log 2>&1
timeout 120 python tools/ptrace.py c4 > $O/ptrace.log 2>&1
cat $O/rc.txt; grep -v "^\[lrs\]" $O/ablate_c4.log
