mkdir -p gpurun_out/r02p1; O=gpurun_out/r02p1
timeout 60 ./tools/probe_2cta 0 > $O/mode0.log 2>&1; echo "rc0=$?" >> $O/mode0.log
timeout 60 ./tools/probe_2cta 1 > $O/mode1.log 2>&1; echo "rc1=$?" >> $O/mode1.log
cat $O/mode0.log $O/mode1.log
