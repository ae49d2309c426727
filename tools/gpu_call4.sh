mkdir -p gpurun_out; rm -f gpurun_out/probe4.log
for a in "128 0 4 2" "128 0 4 4" "128 1 4 2" "128 1 4 4"; do timeout 30 ./tools/sp_probe4 $a >> gpurun_out/probe4.log 2>&1; done
cat gpurun_out/probe4.log
