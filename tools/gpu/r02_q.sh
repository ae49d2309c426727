mkdir -p gpurun_out/r02q; O=gpurun_out/r02q
timeout 300 python -m pytest tests/test_gpu_bounds.py -q > $O/pytest_bounds.log 2>&1; echo "bounds rc=$?" > $O/rc.txt
timeout 2400 python tools/f2_speed_bound.py > $O/f2.log 2>&1; echo "f2 rc=$?" >> $O/rc.txt
cp profiles/r02_f2_speed_bound.json $O/ 2>/dev/null
cat $O/rc.txt; tail -3 $O/pytest_bounds.log; tail -12 $O/f2.log
