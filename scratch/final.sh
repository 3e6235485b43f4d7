cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
TAG=${TAG:-v6}
{
echo "== pytest"; timeout 1200 python -m pytest tests -m gpu -q -rs 2>&1 | tail -4
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
echo "== bench"; timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo rc=$?; tail -2 gpurun_out/${TAG}_bench.err
cat gpurun_out/${TAG}_bench.json
echo "== bench fp32"; timeout 900 python bench.py --precision 32 --no-cpu > gpurun_out/${TAG}_bench_fp32.json 2>&1; tail -1 gpurun_out/${TAG}_bench_fp32.json
echo "== reference arm"; timeout 600 python bench.py --impl reference --steps 200 --warmup 5 2>&1 | tail -1
} > gpurun_out/${TAG}_final.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-batch64 > /dev/null 2>&1
for k in fwd_cluster inv_cluster gather wfs; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_$k -s 6 -c 1 -o gpurun_out/${TAG}_$k -f python tools/profile_frame.py --frames 2 > /dev/null 2>&1
done
cat gpurun_out/${TAG}_final.log
