python bench.py --steps 200 --warmup 5 --no-batch64 --no-configs --no-cpu > gpurun_out/c8.json 2>/dev/null
FEWHA_CLUSTER_ROWS=8 python bench.py --steps 200 --warmup 5 --no-batch64 --no-configs --no-cpu > gpurun_out/c16.json 2> gpurun_out/c16.err
FEWHA_CLUSTER_ROWS=8 python tools/graph_timeline.py 2>&1 | tail -6
FEWHA_CLUSTER_ROWS=8 python -m pytest tests/test_gpu_parity.py -q -x -k "operators or closed_loop" 2>&1 | tail -3
for f in c8 c16; do python -c "
import json; j=json.load(open('gpurun_out/$f.json')); print('$f', 'lat',j['latency']['p50_ms'],j['latency']['p99_ms'], {k:v['launch_ms'] for k,v in j['roofline']['functions'].items()})"; done
tail -3 gpurun_out/c16.err
