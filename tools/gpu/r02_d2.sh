mkdir -p gpurun_out/r02d2; O=gpurun_out/r02d2
LRS_VERBOSE=1 timeout 300 python tools/ablate.py c3 base "LRS_WCONV_ERING=1" "LRS_WCONV_ERING=1 LRS_WCONV_EPI=direct" "LRS_WCONV_ERING=1 LRS_WCONV_EPI=direct LRS_WCONV_NS=2" > $O/ablate_c3.log 2>&1
grep "wconv plan\|c3 \[\|rror" $O/ablate_c3.log
