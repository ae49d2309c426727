mkdir -p gpurun_out/r02p6; O=gpurun_out/r02p6
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 "LRS_WCONV_PAIR=1 LRS_WCONV_BPI=2" "LRS_WCONV_PAIR=1 LRS_WCONV_BPI=2 LRS_WCONV_NS=3" "LRS_WCONV_PAIR=1 LRS_WCONV_NWB1=1" "LRS_WCONV_PAIR=1 LRS_WCONV_BPI=2 LRS_WCONV_NWB1=1" > $O/ablate_c3.log 2>&1
grep "wconv plan\|c3 \[" $O/ablate_c3.log
