mkdir -p gpurun_out/r02p9; O=gpurun_out/r02p9
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "gpu rc=$?" > $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -3 $O/pytest_gpu.log; tail -8 $O/smoke.log
