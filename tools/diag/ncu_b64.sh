# ncu --set full of the batch-64 per-WFS / gather / forward / inverse kernels (one launch each)
P="python tools/profile_frame.py --batch 64 --frames 1"
ncu --set full --clock-control none --import-source on -k regex:k_wfs -s 11 -c 1 -o gpurun_out/b64_wfs $P > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gather -s 11 -c 1 -o gpurun_out/b64_gather $P > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fwd -s 11 -c 1 -o gpurun_out/b64_fwd $P > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_inv -s 11 -c 1 -o gpurun_out/b64_inv $P > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 42 -c 21 --csv --log-file gpurun_out/b64_launches.csv $P > /dev/null 2>&1
ls -la gpurun_out
