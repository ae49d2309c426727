mkdir -p gpurun_out
timeout 120 ./tools/sp_probe3 1 0 > gpurun_out/probe3_sel1.log 2>&1; echo rc=$?
timeout 120 ./tools/sp_probe3 0 0 > gpurun_out/probe3_sel0.log 2>&1; echo rc=$?
tail -3 gpurun_out/probe3_sel1.log gpurun_out/probe3_sel0.log
