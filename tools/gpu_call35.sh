mkdir -p gpurun_out; rm -f gpurun_out/rc35.txt
timeout 900 python -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_parity.py tests/test_gpu_core_fused.py tests/test_gpu_cp.py tests/test_gpu_c5.py -q -x > gpurun_out/pytest_35.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc35.txt
for c in c4 c2_bf16 c3; do
 for cp in 0; do
  r=$(LRS_WCONV_CPW=$cp LRS_VERBOSE=1 timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e 2>gpurun_out/b35.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), round(d['value']))")
  echo "$c cpw_env=$cp $r $(grep 'wconv plan' gpurun_out/b35.err | head -1)" >> gpurun_out/rc35.txt
 done
done
cat gpurun_out/rc35.txt
