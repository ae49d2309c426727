mkdir -p gpurun_out/r02u; O=gpurun_out/r02u
LRS_VERBOSE=1 timeout 600 python tools/ablate.py c3 "LRS_WCONV_IPW=8 LRS_WCONV_TH=7" "LRS_WCONV_IPW=4 LRS_WCONV_BPI=2" "LRS_WCONV_IPW=4 LRS_WCONV_BPI=2 LRS_WCONV_NS=4" "LRS_WCONV_IPW=4 LRS_WCONV_TH=4" "LRS_WCONV_IPW=4 LRS_WCONV_BPI=2 LRS_WCONV_TH=4" > $O/ablate_c3.log 2>&1
LRS_VERBOSE=1 timeout 600 python tools/ablate.py c2_bf16 "LRS_WCONV_IPW=8 LRS_WCONV_TH=7" "LRS_WCONV_IPW=8 LRS_WCONV_TH=4" "LRS_WCONV_IPW=4 LRS_WCONV_BPI=2" "LRS_WCONV_IPW=4 LRS_WCONV_TH=7" "LRS_WCONV_IPW=4 LRS_WCONV_TH=4 LRS_WCONV_BPI=2" > $O/ablate_c2.log 2>&1
LRS_VERBOSE=1 timeout 600 python tools/ablate.py c4 "LRS_NO_PW=1 LRS_WCONV_IPW=8" "LRS_NO_PW=1 LRS_WCONV_IPW=4" > $O/ablate_c4.log 2>&1
grep -h "\] \|wconv plan" $O/ablate_c3.log $O/ablate_c2.log $O/ablate_c4.log | grep -v "\[lrs\] core\|autotune"
