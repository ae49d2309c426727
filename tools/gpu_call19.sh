mkdir -p gpurun_out; rm -f gpurun_out/rc19.txt
timeout 900 python -m pytest tests/test_gpu_core_fused.py -q -x > gpurun_out/pytest_core.log 2>&1; echo "pytest core rc=$?" >> gpurun_out/rc19.txt
python tools/ctrace.py c2_bf16 >> gpurun_out/rc19.txt 2>&1
for c in c2_bf16 c3; do
  for ipt in 0 1 2; do
    r=$(LRS_VERBOSE=1 LRS_CORE_IPT=$ipt timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e 2>gpurun_out/b19_$c.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2), d['roofline']['stage_us'])")
    echo "$c ipt=$ipt $r $(grep core: gpurun_out/b19_$c.err)" >> gpurun_out/rc19.txt
  done
done
cat gpurun_out/rc19.txt
