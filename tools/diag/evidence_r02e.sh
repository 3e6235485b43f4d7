# round-2 (fourth session) evidence: GPU tests, smoke, bench lines (fp64, fp32), graph
# timeline, launch lists (single frame, batch 64), ncu of the dominant kernels
set -u
mkdir -p gpurun_out
python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/e_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.txt 2>&1
python bench.py > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
python bench.py --precision 32 --no-cpu > gpurun_out/r02e_bench_fp32.json 2> gpurun_out/r02e_bench_fp32.err
python tools/graph_timeline.py > gpurun_out/r02e_graph_timeline.txt 2>&1
P1="python tools/profile_frame.py --frames 1"
P64="python tools/profile_frame.py --batch 64 --frames 1"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
ncu $M -s 42 -c 21 --log-file gpurun_out/r02e_launches_b1.csv $P1 > /dev/null 2>&1
ncu $M -s 42 -c 21 --log-file gpurun_out/r02e_launches_b64.csv $P64 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_inv_cluster -s 11 -c 1 -o gpurun_out/r02e_inv_b1 $P1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_inv_layer -s 12 -c 1 -o gpurun_out/r02e_inv_b64 $P64 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gather_direct -s 12 -c 1 -o gpurun_out/r02e_gather_b64 $P64 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gather_direct -s 11 -c 1 -o gpurun_out/r02e_gather_b1 $P1 > /dev/null 2>&1
cat gpurun_out/e_tests.txt gpurun_out/e_smoke.txt
ls gpurun_out | grep r02e
ncu --set full --import-source on --clock-control none -k regex:k_wfs -s 6 -c 1 -o gpurun_out/r02e_wfs_b64 $P64 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_wfs -s 5 -c 1 -o gpurun_out/r02e_wfs_b1 $P1 > /dev/null 2>&1
ls gpurun_out | grep r02e
# keep the merge under 64 MiB: export the captures' pages and drop the reports
for r in gpurun_out/r02e_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page details --csv > ${b}_details.csv 2>/dev/null
  ncu -i $r --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > ${b}_source.csv 2>/dev/null
  rm -f $r
done
du -sh gpurun_out
