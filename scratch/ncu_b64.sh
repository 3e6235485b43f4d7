cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for k in wfs gather inv_cluster fwd_cluster; do
  timeout 600 $NCU --set full --clock-control none -k regex:k_$k -s 6 -c 1 -o gpurun_out/b64_$k -f python tools/profile_frame.py --batch 64 --frames 1 > gpurun_out/b64_ncu_$k.log 2>&1
  tail -1 gpurun_out/b64_ncu_$k.log
done
