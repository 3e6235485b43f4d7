cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -x -q -rs 2>&1 | tail -15
timeout 300 python scratch/timing.py 2>&1 | tail -12
timeout 300 python scratch/stamps2.py 2>&1 | tail -12
} > gpurun_out/perf.log 2>&1
cat gpurun_out/perf.log
