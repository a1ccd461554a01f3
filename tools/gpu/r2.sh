timeout 1700 python -m pytest tests/test_gpu_configs.py -q -m gpu --durations=10 > gpurun_out/t_configs.log 2>&1
echo rc=$?
