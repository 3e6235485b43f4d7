# A/B: WFS tile kernel with four (default) vs eight instances per CTA (batch 64)
set -u
for p in 64 32; do
  for n in 4 8 4 8; do
    echo "fp$p ni $n: $(FEWHA_WFS_NI=$n timeout 300 python tools/diag/ab_lat.py --batch 64 --precision $p --frames 200 2>&1 | tail -1)"
  done
done
echo "fp32 8x8 ni 8:"; FEWHA_WFS_NI=8 timeout 300 python tools/batch_sweep.py --sizes 8 --precision 32 2>&1 | grep concurrent
echo "fp32 8x8 ni 4:"; timeout 300 python tools/batch_sweep.py --sizes 8 --precision 32 2>&1 | grep concurrent
