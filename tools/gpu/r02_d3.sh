mkdir -p gpurun_out/r02d3; O=gpurun_out/r02d3
timeout 300 python tools/ablate.py c3 base "CFG_density=0.02" "CFG_density=0.01" "CFG_density=0.0" "CFG_density=0.1" > $O/ablate_c3.log 2>&1
timeout 300 python tools/ablate.py c2_bf16 base "CFG_density=0.02" "CFG_density=0.0" > $O/ablate_c2.log 2>&1
cat $O/*.log | grep "\[\|rror"
