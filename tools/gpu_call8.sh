mkdir -p gpurun_out; rm -f gpurun_out/rc8.txt
python -c "from paper_2006_06443_b200 import _build as b; print(b.needs_build())" > gpurun_out/needs_build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_spadd_f32.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_spadd.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc8.txt
for c in c2_f32 c1; do
  LRS_VERBOSE=1 timeout 600 python bench.py --config $c --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/rc8.txt
done
timeout 120 python tools/gpu_debug.py c2_bf16 > gpurun_out/plain_c2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -c 2 -o gpurun_out/prof_gemm_c2 python tools/gpu_debug.py c2_bf16 > gpurun_out/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?" >> gpurun_out/rc8.txt
timeout 120 python tools/gpu_debug.py c2_f32 > gpurun_out/plain_c2f.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spadd -c 1 -o gpurun_out/prof_spadd_c2 python tools/gpu_debug.py c2_f32 > gpurun_out/ncu_spadd.log 2>&1; echo "ncu spadd rc=$?" >> gpurun_out/rc8.txt
cat gpurun_out/rc8.txt
