# round 2, call E: ncu of the pw kernel at C4; C3 one-block-item plans
mkdir -p gpurun_out/r02e; O=gpurun_out/r02e
timeout 120 python tools/run_layer.py c4 4 > $O/plain_c4.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lrs_pw -s 2 -c 1 -o $O/prof_pw_c4 -f python tools/run_layer.py c4 4 > $O/ncu_pw_c4.log 2>&1; echo "ncu rc=$?" > $O/rc.txt
timeout 300 python tools/ablate.py c3 base "LRS_WCONV_BPI=1 LRS_WCONV_NS=6" "LRS_WCONV_BPI=1 LRS_WCONV_NS=5" "LRS_WCONV_BPI=1 LRS_WCONV_NS=4" > $O/ablate_c3.log 2>&1; echo "abl rc=$?" >> $O/rc.txt
timeout 300 python tools/ablate.py c4 base "LRS_PW_MPC=2 LRS_PW_BP=112" "LRS_PW_MPC=2 LRS_PW_BP=96" "LRS_PW_MPC=4 LRS_PW_BP=64" "LRS_NO_PW=1" > $O/ablate_c4.log 2>&1; echo "abl4 rc=$?" >> $O/rc.txt
cat $O/rc.txt
