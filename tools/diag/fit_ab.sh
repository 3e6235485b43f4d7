# fit kernel with 4 pre-wait layer stencils (40 / 59 registers instead of 128): latency + batch, tests
set -u
mkdir -p gpurun_out
for k in 1 2; do
  echo "single: $(timeout 300 python tools/diag/ab_lat.py --frames 600 2>&1 | tail -1)" >> gpurun_out/fit_ab.txt
  echo "b64 fp64: $(timeout 300 python tools/diag/ab_lat.py --batch 64 --frames 200 2>&1 | tail -1)" >> gpurun_out/fit_ab.txt
done
timeout 300 python tools/diag/batch_funcs.py >> gpurun_out/fit_ab.txt 2>&1
timeout 1200 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_plans.py tests/test_gpu_dropin.py 2>&1 | tail -2 >> gpurun_out/fit_ab.txt
cat gpurun_out/fit_ab.txt
