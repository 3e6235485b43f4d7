python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_plans.py -q -x 2>&1 | tail -2
python tools/diag/ab.py "{}"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -s 42 -c 21 --log-file gpurun_out/gat_b1.csv python tools/profile_frame.py --frames 1 > /dev/null 2>&1
python tools/dram_traffic.py x=gpurun_out/gat_b1.csv
