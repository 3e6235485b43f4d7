# ncu --set full of the WFS tile kernel and the whole-layer forward, batch 64 (fp64)
set -u
mkdir -p gpurun_out
P64="python tools/profile_frame.py --batch 64 --frames 1"
ncu --set full --import-source on --clock-control none -k regex:k_wfs -s 6 -c 1 -o gpurun_out/r02e_wfs_b64 $P64 > gpurun_out/ncu_wfs.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fwd_layer -s 3 -c 1 -o gpurun_out/r02e_fwd_b64 $P64 > gpurun_out/ncu_fwd.log 2>&1
ls -la gpurun_out
