mkdir -p gpurun_out/r02g2; O=gpurun_out/r02g2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lrs_wconv -s 2 -c 1 -o $O/prof_wconv_c3 -f python tools/run_layer.py c3 4 > $O/ncu.log 2>&1; echo "ncu rc=$?"
tail -3 $O/ncu.log
