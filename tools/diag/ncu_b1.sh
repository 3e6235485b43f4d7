P="python tools/profile_frame.py --frames 1"
ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:k_fwd_cluster -s 11 -c 1 -o gpurun_out/b1_fwd $P > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:k_inv_cluster -s 11 -c 1 -o gpurun_out/b1_inv $P > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
