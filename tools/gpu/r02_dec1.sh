# decomposition (f4): GPU tests
mkdir -p gpurun_out/dec1; O=gpurun_out/dec1; rm -f $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_decomp.py -q -x > $O/pytest_dec.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
cat $O/rc.txt
