mkdir -p gpurun_out/r02e6; O=gpurun_out/r02e6
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c4 base "LRS_PW_MPC=2 LRS_PW_BP=128 LRS_PW_CPI=1" "LRS_PW_MPC=2 LRS_PW_BP=128 LRS_PW_CPI=2" "LRS_PW_MPC=1 LRS_PW_BP=128 LRS_PW_CPI=1" "LRS_PW_MPC=2 LRS_PW_BP=96 LRS_PW_CPI=2" "LRS_PW_MPC=1 LRS_PW_BP=96 LRS_PW_CPI=2" "LRS_PW_MPC=2 LRS_PW_BP=64 LRS_PW_CPI=4" > $O/ablate_c4.log 2>&1
grep "pw plan\|c4 \[" $O/ablate_c4.log
