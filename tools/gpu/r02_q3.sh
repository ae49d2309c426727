mkdir -p gpurun_out/r02q3; O=gpurun_out/r02q3
LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
E="LRS_SKIP=1 LRS_PW_MPC=2 LRS_PW_BP=96 LRS_PW_CPI=2"
timeout 300 python tools/ablate.py c4 "$E" "$E LRS_PW_DBG=1" "$E LRS_PW_DBG=9" "$E LRS_PW_DBG=25" "$E LRS_PW_DBG=57" "$E LRS_PW_DBG=7" "$E LRS_PW_DBG=63" "$E LRS_PW_DBG=6" > $O/ablate.log 2>&1
grep "c4 \[" $O/ablate.log
