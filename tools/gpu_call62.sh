mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse_tc.py tests/test_gpu_epilogue.py -q > gpurun_out/t62.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/t62.log
for c in c2_bf16 c3 c4; do
timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b62_$c.json 2> gpurun_out/b62_$c.err; echo "$c rc=$?"; tail -1 gpurun_out/b62_$c.json | cut -c140-200
done
LRS_WCONV_REUSE=1 timeout 300 python bench.py --config c4 --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/b62_c4r.json 2> gpurun_out/b62_c4r.err; echo "c4 reuse rc=$?"; tail -1 gpurun_out/b62_c4r.json | cut -c140-200
LRS_WCONV_DEBUG=1 python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
timeout 120 python tools/wtrace.py c2_bf16 > gpurun_out/wtrace62_c2.log 2>&1
timeout 120 python tools/wtrace.py c4 > gpurun_out/wtrace62_c4.log 2>&1
python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
head -3 gpurun_out/wtrace62_c2.log; head -8 gpurun_out/wtrace62_c4.log
