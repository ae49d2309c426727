mkdir -p gpurun_out/r02p7; O=gpurun_out/r02p7
timeout 120 ./tools/probe_2cta_rate > $O/rate.log 2>&1; echo "rc=$?" >> $O/rate.log
cat $O/rate.log
