set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -m gpu --durations=10 > gpurun_out/t_configs.log 2>&1
echo rc=$?
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --timesteps 20 > gpurun_out/b_c3.log 2>&1
echo rc=$?
lscpu | head -20 > gpurun_out/lscpu.txt
