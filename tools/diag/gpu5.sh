python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/t_all.txt
python bench.py --steps 20 --warmup 5 --no-batch64 --no-configs --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
cat gpurun_out/t_all.txt; python -c "
import json; j=json.load(open('gpurun_out/bench_quick.json')); print('p50',j['p50_ms'],'lat',j['latency']['p50_ms'],j['latency']['p99_ms'],'e2e',j['e2e']['p50_ms'], j['roofline']['functions'])"
