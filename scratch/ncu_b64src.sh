cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for k in wfs gather; do
  timeout 600 $NCU --set full --import-source on --clock-control none -k regex:k_$k -s 6 -c 1 -o gpurun_out/b64s_$k -f python tools/profile_frame.py --batch 64 --frames 1 > /dev/null 2>&1
done
ls gpurun_out/b64s_*
