# A/B: WFS tile kernel with four instances per CTA at 4 vs 6 CTAs per SM (batch 64)
set -u
mkdir -p gpurun_out
for p in 64 32; do
  echo "fp$p ni4 4/SM: $(timeout 300 python tools/diag/ab_lat.py --batch 64 --precision $p --frames 200 2>&1 | tail -1)" >> gpurun_out/wn_ab.txt
  echo "fp$p ni4 6/SM: $(FEWHA_WFS_NI4_6=1 timeout 300 python tools/diag/ab_lat.py --batch 64 --precision $p --frames 200 2>&1 | tail -1)" >> gpurun_out/wn_ab.txt
  echo "fp$p ni4 4/SM: $(timeout 300 python tools/diag/ab_lat.py --batch 64 --precision $p --frames 200 2>&1 | tail -1)" >> gpurun_out/wn_ab.txt
  echo "fp$p ni4 6/SM: $(FEWHA_WFS_NI4_6=1 timeout 300 python tools/diag/ab_lat.py --batch 64 --precision $p --frames 200 2>&1 | tail -1)" >> gpurun_out/wn_ab.txt
done
timeout 600 python -m pytest -q -x tests/test_gpu_plans.py 2>&1 | tail -2 >> gpurun_out/wn_ab.txt
cat gpurun_out/wn_ab.txt
