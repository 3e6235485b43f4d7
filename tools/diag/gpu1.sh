set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
python tools/diag/loop_errors.py elt_mcao84 30 64 > gpurun_out/d_elt64.txt 2>&1
python tools/diag/loop_errors.py elt_mcao84 30 32 > gpurun_out/d_elt32.txt 2>&1
python tools/diag/loop_errors.py small_mcao 12 32 > gpurun_out/d_small32.txt 2>&1
python tools/diag/loop_errors.py elt_mcao84_3dm 10 64 4 > gpurun_out/d_b4_64.txt 2>&1
python tools/diag/loop_errors.py elt_mcao84_3dm 10 32 4 > gpurun_out/d_b4_32.txt 2>&1
FEWHA_TAIL=16 FEWHA_INV_STAGE=0 python tools/diag/loop_errors.py elt_mcao84_3dm 10 64 1 > gpurun_out/d_b1knob_64.txt 2>&1
tail -3 gpurun_out/d_*.txt
