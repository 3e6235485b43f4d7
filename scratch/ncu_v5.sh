cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
TAG=${TAG:-v5}
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-batch64 > gpurun_out/${TAG}_launch_bench.log 2>&1
for k in fwd_cluster inv_cluster gather wfs; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_$k -s 6 -c 1 -o gpurun_out/${TAG}_$k -f python tools/profile_frame.py --frames 2 > gpurun_out/${TAG}_ncu_$k.log 2>&1
  tail -2 gpurun_out/${TAG}_ncu_$k.log
done
ls -la gpurun_out
