#!/bin/bash
# full capture of the config-4 packed element kernel (one 512-column batch)
cd "$(dirname "$0")/../.."
LSB_ELEM_F2=1 ncu --set full --clock-control none --import-source on -k regex:elem_batched_p2 -s 2 -c 1 -o gpurun_out/p2_c4 -f python tools/batched_timing.py 1024 1 > gpurun_out/ncu_p2.log 2>&1
python tools/ncu_report.py gpurun_out/p2_c4.ncu-rep > gpurun_out/p2_c4.txt
head -50 gpurun_out/p2_c4.txt
