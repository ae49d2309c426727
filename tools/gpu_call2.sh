mkdir -p gpurun_out; rm -f gpurun_out/probe2.log
for pm in 1 2 3 4; do
 for h in 10 11 12 13 14 15 0 2; do echo -n "pmode $pm: " >> gpurun_out/probe2.log; timeout 30 ./tools/sp_probe2 $h $pm 2>&1 | grep -v BEST >> gpurun_out/probe2.log; done
done
cat gpurun_out/probe2.log
