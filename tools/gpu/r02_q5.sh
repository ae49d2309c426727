mkdir -p gpurun_out/r02q5; O=gpurun_out/r02q5
timeout 600 python -m pytest $(grep -ln "forward_host" tests/test_gpu*.py) -x -q > $O/pytest.log 2>&1; echo "rc=$?" > $O/rc.txt
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu --no-dense > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench rc=$?" >> $O/rc.txt
timeout 600 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu --no-dense > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc=$?" >> $O/rc.txt
cat $O/rc.txt; tail -2 $O/pytest.log; python -c "
import json
for c in ('c3','c4'):
    d=json.loads(open('$O/bench_'+c+'.json').read().strip().splitlines()[-1]); print(c, round(d['value']), 'e2e', round(d['e2e']['value']), d['verify'].get('e2e_bitwise_device_forward'))"
