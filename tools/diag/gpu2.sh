python -m pytest tests/test_gpu_plans.py -x -q -s 2>&1 | tail -25 > gpurun_out/t_plans.txt
python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/t_all.txt
cat gpurun_out/t_plans.txt gpurun_out/t_all.txt
