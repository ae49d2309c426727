mkdir -p gpurun_out
timeout 600 python bench.py --config c2_bf16 --steps 200 --warmup 10 > gpurun_out/bench66_c2_bf16.json 2> gpurun_out/bench66_c2_bf16.err; echo "c2 rc=$?"
timeout 300 python bench.py > gpurun_out/bench66_default.json 2> gpurun_out/bench66_default.err; echo "default rc=$?"
tail -1 gpurun_out/bench66_default.json | cut -c1-300
