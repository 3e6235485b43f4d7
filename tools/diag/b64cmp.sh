python bench.py --steps 50 --warmup 5 --no-configs --no-cpu --precision 64 > gpurun_out/p64.json 2>/dev/null
python bench.py --steps 50 --warmup 5 --no-configs --no-cpu --precision 32 > gpurun_out/p32.json 2>/dev/null
python -m pytest tests/test_gpu_parity.py tests/test_gpu_plans.py -q -x -k "32" 2>&1 | tail -3
for f in p64 p32; do python -c "
import json; j=json.load(open('gpurun_out/$f.json')); b=j['batch64']; print('$f', 'lat',j['latency']['p50_ms'], 'b64 ms',b['ms_per_step'],'rps',b['recon_per_s'],'frac',b['roofline_frac_frame_model'], {k:v['launch_ms'] for k,v in b['roofline']['functions'].items()})"; done
