mkdir -p gpurun_out/r02x; O=gpurun_out/r02x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_parity.log 2>&1; echo "parity rc=$?" > $O/rc.txt
timeout 2400 python tools/f2_speed_bound.py > $O/f2.log 2>&1; echo "f2 rc=$?" >> $O/rc.txt
cp profiles/r02_f2_speed_bound.json $O/ 2>/dev/null
cat $O/rc.txt; tail -3 $O/pytest_parity.log; grep "^x3 L [1-9]\|^x3 L1[01]" $O/f2.log | head -12; tail -12 $O/f2.log
