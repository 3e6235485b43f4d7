cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/profile_frame.py --batch 64 --frames 3 2>&1 | tail -3
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__shared_mem_per_block_dynamic,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__cluster_max_active_clusters --clock-control none -s 42 -c 21 --csv --log-file gpurun_out/b64_launches.csv python tools/profile_frame.py --batch 64 --frames 1 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(l for l in open('gpurun_out/b64_launches.csv') if l.startswith('"')))
h=rows[0]; per=collections.OrderedDict()
for r in rows[1:]:
    d=dict(zip(h,r)); k=(d['ID'], d['Kernel Name'][:40]); per.setdefault(k,{})[d['Metric Name']]=d['Metric Value']
for k,v in per.items(): print(k, {m.split('.')[0].replace('launch__','').replace('gpu__',''):x for m,x in v.items()})
PY
