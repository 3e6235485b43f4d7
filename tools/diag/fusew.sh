# A/B of the fused whole-layer forward + inverse (k_fwd_inv_layer) for batches
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_plans.py tests/test_gpu_parity.py -k "whole or batch or fused" 2>&1 | tail -15 > gpurun_out/fw_tests.txt
for p in 64 32; do
  for f in 0 1; do
    echo "prec $p fuse $f: $(FEWHA_FUSE_WHOLE=$f timeout 300 python tools/diag/ab_lat.py --batch 64 --precision $p --frames 200 2>&1 | tail -1)" >> gpurun_out/fw_ab.txt
  done
done
FEWHA_FUSE_WHOLE=1 timeout 300 python tools/diag/batch_funcs.py > gpurun_out/fw_funcs.txt 2>&1
cat gpurun_out/fw_tests.txt gpurun_out/fw_ab.txt
