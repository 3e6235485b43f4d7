# round-2 (fourth session, final state after the fit kernel change) evidence: GPU tests, smoke, bench lines (fp64, fp32),
# batch-64 launch list and the WFS kernel capture of the final plan
set -u
mkdir -p gpurun_out
python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/g_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.txt 2>&1
python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
python bench.py --precision 32 --no-cpu > gpurun_out/r02g_bench_fp32.json 2> gpurun_out/r02g_bench_fp32.err
P64="python tools/profile_frame.py --batch 64 --frames 1"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
ncu $M -s 42 -c 21 --log-file gpurun_out/r02g_launches_b64.csv $P64 > /dev/null 2>&1
ncu $M -s 42 -c 21 --log-file gpurun_out/r02g_launches_b1.csv python tools/profile_frame.py --frames 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_wfs -s 6 -c 1 -o gpurun_out/r02g_wfs_b64 $P64 > /dev/null 2>&1
ncu -i gpurun_out/r02g_wfs_b64.ncu-rep --page details --csv > gpurun_out/r02g_wfs_b64_details.csv 2>/dev/null
ncu -i gpurun_out/r02g_wfs_b64.ncu-rep --page raw --csv > gpurun_out/r02g_wfs_b64_raw.csv 2>/dev/null
rm -f gpurun_out/r02g_wfs_b64.ncu-rep
cat gpurun_out/g_tests.txt gpurun_out/g_smoke.txt
