mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_core_fused.py tests/test_gpu_parity.py -q -x > gpurun_out/t53.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/t53.log
timeout 900 python tools/core_sweep.py c2_bf16 1,7 1,7,36 1,14 1,14,36 2,7,36 > gpurun_out/core_sweep53_c2.log 2>&1; echo "sweep rc=$?"
timeout 900 python tools/core_sweep.py c3 1,7 2,7 1,7,64 > gpurun_out/core_sweep53_c3.log 2>&1; echo "sweep c3 rc=$?"
LRS_WCONV_DEBUG=1 python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
for v in "1,7,148" "1,7,36" "1,14,36" "1,7,16"; do
  export LRS_CORE_IPT=$(echo $v | cut -d, -f1) LRS_CORE_TH=$(echo $v | cut -d, -f2) LRS_CORE_GRID=$(echo $v | cut -d, -f3)
  echo "== ipt,th,grid=$v" >> gpurun_out/ctrace53_c2.log
  timeout 120 python tools/ctrace.py c2_bf16 >> gpurun_out/ctrace53_c2.log 2>&1
done
unset LRS_CORE_IPT LRS_CORE_TH LRS_CORE_GRID
timeout 120 python tools/ctrace.py c3 > gpurun_out/ctrace53_c3.log 2>&1
python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
