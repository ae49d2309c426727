mkdir -p gpurun_out
LRS_WCONV_DEBUG=1 python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
for v in "1,7,148" "1,7,36" "2,7,36"; do
  export LRS_CORE_IPT=$(echo $v | cut -d, -f1) LRS_CORE_TH=$(echo $v | cut -d, -f2) LRS_CORE_GRID=$(echo $v | cut -d, -f3)
  echo "== ipt,th,grid=$v" >> gpurun_out/ctrace61_c2.log
  timeout 120 python tools/ctrace.py c2_bf16 >> gpurun_out/ctrace61_c2.log 2>&1
done
unset LRS_CORE_IPT LRS_CORE_TH LRS_CORE_GRID
timeout 120 python tools/wtrace.py c2_bf16 > gpurun_out/wtrace61_c2.log 2>&1
python -m paper_2006_06443_b200._build --force > /dev/null 2>&1
cat gpurun_out/ctrace61_c2.log
