# round 2, call D: the channel-stationary 1x1 kernel (C4)
mkdir -p gpurun_out/r02d; O=gpurun_out/r02d
LRS_VERBOSE=1 timeout 300 python -m pytest tests/test_gpu_pw.py -x -q > $O/pytest_pw.log 2>&1; echo "pw rc=$?" > $O/rc.txt
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "gpu rc=$?" >> $O/rc.txt
timeout 300 python bench.py --config c4 --steps 200 --warmup 10 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench rc=$?" >> $O/rc.txt
LRS_VERBOSE=1 timeout 120 python -c "
import workloads
from paper_2006_06443_b200 import LrsConv
LrsConv.from_inputs(workloads.generate(workloads.CONFIGS['c4'], batch=1), batch_max=128)" > $O/plan_c4.log 2>&1
cat $O/rc.txt
