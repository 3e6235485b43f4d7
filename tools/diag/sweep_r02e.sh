# engines x instances per step (64 total) on concurrent streams, fp64 / fp32, after the WFS change
set -u
mkdir -p gpurun_out
timeout 600 python tools/batch_sweep.py --sizes 8,16,32,64 --precision 64 > gpurun_out/sw64.txt 2>&1
timeout 600 python tools/batch_sweep.py --sizes 8,16,32,64 --precision 32 > gpurun_out/sw32.txt 2>&1
timeout 600 python -m pytest -q -x tests/test_gpu_plans.py 2>&1 | tail -2 > gpurun_out/sw_tests.txt
cat gpurun_out/sw64.txt gpurun_out/sw32.txt gpurun_out/sw_tests.txt
