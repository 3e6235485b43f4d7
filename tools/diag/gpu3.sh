python -m pytest tests/test_gpu_plans.py tests/test_gpu_properties.py -q -s 2>&1 | tail -40 > gpurun_out/t_new.txt
cat gpurun_out/t_new.txt
