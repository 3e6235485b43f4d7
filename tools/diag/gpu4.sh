P1="python tools/profile_frame.py --frames 1"
P64="python tools/profile_frame.py --batch 64 --frames 1"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
ncu $M -s 42 -c 21 --log-file gpurun_out/r02_launches_b1.csv $P1 > /dev/null 2>&1
ncu $M -s 42 -c 21 --log-file gpurun_out/r02_launches_b64.csv $P64 > /dev/null 2>&1
python tools/dram_traffic.py fp64=gpurun_out/r02_launches_b1.csv fp64_b64=gpurun_out/r02_launches_b64.csv
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -3 gpurun_out/bench_quick.err
cp profiles/dram_traffic.json gpurun_out/
