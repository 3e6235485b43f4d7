# A/B: WFS tile kernel residency / instances per CTA (batch 64)
set -u
mkdir -p gpurun_out
for m in 5 6 5 6; do
  echo "fp64 ni2 minb $m: $(FEWHA_WFS_NI2_MINB=$m timeout 300 python tools/diag/ab_lat.py --batch 64 --precision 64 --frames 200 2>&1 | tail -1)" >> gpurun_out/wm_ab.txt
done
for m in 2 4 2 4; do
  echo "fp32 ni4 minb $m: $(FEWHA_WFS_NI4_MINB=$m timeout 300 python tools/diag/ab_lat.py --batch 64 --precision 32 --frames 200 2>&1 | tail -1)" >> gpurun_out/wm_ab.txt
done
echo "fp32 ni2 minb 6: $(FEWHA_WFS_NI=2 FEWHA_WFS_NI2_MINB=6 timeout 300 python tools/diag/ab_lat.py --batch 64 --precision 32 --frames 200 2>&1 | tail -1)" >> gpurun_out/wm_ab.txt
cat gpurun_out/wm_ab.txt
