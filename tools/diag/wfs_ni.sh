# A/B: fp64 WFS tile kernel with two (6/SM) vs four (4/SM) instances per CTA (batch 64)
set -u
mkdir -p gpurun_out
for n in 2 4 2 4; do
  echo "fp64 ni $n: $(FEWHA_WFS_NI=$n timeout 300 python tools/diag/ab_lat.py --batch 64 --precision 64 --frames 200 2>&1 | tail -1)" >> gpurun_out/wn_ab.txt
done
cat gpurun_out/wn_ab.txt
