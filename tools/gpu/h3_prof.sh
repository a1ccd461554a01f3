#!/bin/bash
# launch list + full capture of the config-5 element Hessian kernel (64 pairs = 2 chunks)
cd "$(dirname "$0")/../.."
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c5.csv python tools/hessian_timing.py 64 > gpurun_out/ncu_c5.log 2>&1
python tools/ncu_summary.py gpurun_out/launches_c5.csv > gpurun_out/launches_c5.txt
ncu --set full --clock-control none --import-source on -k regex:elem_hess3 -s 1 -c 1 -o gpurun_out/h3_c5 -f python tools/hessian_timing.py 64 > gpurun_out/ncu_c5b.log 2>&1
python tools/ncu_report.py gpurun_out/h3_c5.ncu-rep > gpurun_out/h3_c5.txt
cat gpurun_out/launches_c5.txt; head -60 gpurun_out/h3_c5.txt
