mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_core_fused.py tests/test_gpu_parity.py -q -x > gpurun_out/t52.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/t52.log
LRS_VERBOSE=1 timeout 300 python bench.py --config c2_bf16 --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b52_c2.json 2> gpurun_out/b52_c2.err; tail -1 gpurun_out/b52_c2.json | cut -c1-200; grep "core:" gpurun_out/b52_c2.err | head -2
LRS_VERBOSE=1 timeout 300 python bench.py --config c3 --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b52_c3.json 2> gpurun_out/b52_c3.err; tail -1 gpurun_out/b52_c3.json | cut -c1-200; grep "core:" gpurun_out/b52_c3.err | head -2
timeout 900 python tools/core_sweep.py c2_bf16 1,7 1,7,36 1,7,32 1,7,24 2,14 2,14,16 1,14 1,14,32 1,14,36 2,7,36 1,4,36 2,4,36 4,2,36 2,3,36 1,5,36 > gpurun_out/core_sweep52_c2.log 2>&1; echo "sweep rc=$?"
timeout 900 python tools/core_sweep.py c3 1,7 1,7,64 1,7,48 1,7,36 1,4 1,4,36 2,3,36 1,3,36 > gpurun_out/core_sweep52_c3.log 2>&1; echo "sweep c3 rc=$?"
