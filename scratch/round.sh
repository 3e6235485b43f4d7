cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
echo "== pytest gpu"; timeout 1200 python -m pytest tests -m gpu -x -q -rs 2>&1 | tail -20
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
echo "== bench"; timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$?; tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
echo "== timing"; timeout 300 python scratch/timing.py 2>&1 | tail -12
} > gpurun_out/round.log 2>&1
cat gpurun_out/round.log
