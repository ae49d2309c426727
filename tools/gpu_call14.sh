mkdir -p gpurun_out; rm -f gpurun_out/rc14.txt
timeout 900 python -m pytest tests/test_gpu_core_fused.py -q -x > gpurun_out/pytest_core.log 2>&1; echo "pytest core rc=$?" >> gpurun_out/rc14.txt
for c in c2_bf16 c3; do
  for ipt in 0 1 2; do
    r=$(LRS_VERBOSE=1 LRS_CORE_IPT=$ipt timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e 2>gpurun_out/b14_$c.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), d['roofline']['stage_us'])")
    echo "$c ipt=$ipt $r $(grep core: gpurun_out/b14_$c.err)" >> gpurun_out/rc14.txt
  done
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:core_kernel -c 1 -o gpurun_out/prof_core_c2_bf16 -f python tools/gpu_debug.py c2_bf16 > gpurun_out/ncu_core_c2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/rc14.txt
cat gpurun_out/rc14.txt
