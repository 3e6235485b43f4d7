cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_inv_cluster -s 20 -c 1 -o gpurun_out/inv5 -f python tools/profile_frame.py --frames 4 > /tmp/ncu1.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_fwd_cluster -s 16 -c 1 -o gpurun_out/fwd5 -f python tools/profile_frame.py --frames 4 > /tmp/ncu2.log 2>&1
tail -3 /tmp/ncu1.log /tmp/ncu2.log
ls -la gpurun_out
