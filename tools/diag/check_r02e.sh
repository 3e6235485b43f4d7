# round-2 (fourth session) check: GPU tests, smoke, bench lines (fp64, fp32)
set -u
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x 2>&1 | tail -6 > gpurun_out/e_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.txt 2>&1
python bench.py > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
python bench.py --precision 32 --no-cpu > gpurun_out/r02e_bench_fp32.json 2> gpurun_out/r02e_bench_fp32.err
cat gpurun_out/e_tests.txt gpurun_out/e_smoke.txt
