#!/bin/bash
# Round-2 profile captures (each program first runs once without ncu): launch lists with DRAM bytes and
# --set full captures of the kernels changed this round.  Outputs under gpurun_out/.
cd "$(dirname "$0")/../.."
M3=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python tools/sweep_once.py c3 > gpurun_out/p_c3.log 2>&1 || exit 1
ncu --metrics $M3 --clock-control none -c 40 --csv --log-file gpurun_out/r02_launches_c3.csv python tools/sweep_once.py c3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:elem_kernel -s 1 -c 1 -o gpurun_out/r02_elem_c3 -f python tools/sweep_once.py c3 > /dev/null 2>&1
python tools/hessian_timing.py 128 > gpurun_out/p_c5.log 2>&1 || exit 1
ncu --metrics $M3 --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_c5.csv python tools/hessian_timing.py 128 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:elem_hess3 -s 1 -c 1 -o gpurun_out/r02_elem_hess3_c5 -f python tools/hessian_timing.py 128 > /dev/null 2>&1
python tools/batched_timing.py 512 1 > gpurun_out/p_c4.log 2>&1 || exit 1
ncu --metrics $M3 --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_c4.csv python tools/batched_timing.py 512 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:elem_batched_p2 -s 2 -c 1 -o gpurun_out/r02_elem_p2_c4 -f python tools/batched_timing.py 512 1 > /dev/null 2>&1
python bench.py --records none --steps 3 --warmup 3 --no-cpu-baseline --timesteps 2 > gpurun_out/p_bench.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --records none --steps 3 --warmup 3 --no-cpu-baseline --timesteps 2 > /dev/null 2>&1
for k in elem_c3 elem_hess3_c5 elem_p2_c4; do python tools/ncu_report.py gpurun_out/r02_$k.ncu-rep > gpurun_out/r02_$k.txt; done
ls -la gpurun_out/ | tail -20
