mkdir -p gpurun_out/r02f4; O=gpurun_out/r02f4
LRS_EXPERIMENTS=1 python -m paper_2006_06443_b200._build --force > $O/build.log 2>&1
timeout 300 python tools/ablate.py c2_bf16 base "LRS_CORE_DBG=8" "LRS_CORE_DBG=16" "LRS_CORE_DBG=24" "LRS_CORE_DBG=4" > $O/ablate_c2.log 2>&1
timeout 300 python tools/ablate.py c3 base "LRS_CORE_DBG=8" "LRS_CORE_DBG=16" "LRS_CORE_DBG=24" "LRS_CORE_DBG=4" > $O/ablate_c3.log 2>&1
grep "\[" $O/ablate_c2.log $O/ablate_c3.log
