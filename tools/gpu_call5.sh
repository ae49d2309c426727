set -e; python -c "from paper_2006_06443_b200 import _build; _build.build()"; set +e
mkdir -p gpurun_out; rm -f gpurun_out/dbg5_*.log
for c in "c3 16" "c2_bf16 16" "c4 16" "c3" "c2_bf16" "c4"; do
  tag=${c// /_}; timeout 120 python tools/gpu_debug.py $c > gpurun_out/dbg5_$tag.log 2>&1; echo "$c rc=$?" >> gpurun_out/dbg5_summary.log
done
cat gpurun_out/dbg5_summary.log gpurun_out/dbg5_*.log
