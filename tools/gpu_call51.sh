mkdir -p gpurun_out
./tools/mma_baseoff > gpurun_out/mma_baseoff.log 2>&1; echo "baseoff rc=$?"
timeout 1200 python tools/core_sweep.py c2_bf16 > gpurun_out/core_sweep_c2.log 2>&1; echo "sweep rc=$?"
LRS_WCONV_DEBUG=1 python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
for v in "" "1,7" "2,7" "1,14" "2,2" "4,1" "2,3"; do
  if [ -n "$v" ]; then export LRS_CORE_IPT=${v%%,*} LRS_CORE_TH=${v##*,}; fi
  echo "== ipt,th=$v" >> gpurun_out/ctrace_c2.log
  timeout 120 python tools/ctrace.py c2_bf16 >> gpurun_out/ctrace_c2.log 2>&1
done
unset LRS_CORE_IPT LRS_CORE_TH
timeout 120 python tools/ctrace.py c3 > gpurun_out/ctrace_c3.log 2>&1
python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
timeout 900 python tools/core_sweep.py c3 1,1 1,2 1,3 1,4 1,7 2,1 2,2 2,3 4,1 > gpurun_out/core_sweep_c3.log 2>&1; echo "sweep c3 rc=$?"
