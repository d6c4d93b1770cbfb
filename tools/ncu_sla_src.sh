#!/bin/bash
# ncu source-level capture of the fused attention kernel at cfg4 (one launch)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:sla_tc_kernel -s 1 -c 1 \
    -o gpurun_out/sla_full -f python tools/time_sla.py > gpurun_out/ncu_sla.log 2>&1
ncu -i gpurun_out/sla_full.ncu-rep --page source --csv --print-source sass > gpurun_out/sla_source.csv 2>&1
ncu -i gpurun_out/sla_full.ncu-rep --page raw --csv > gpurun_out/sla_raw.csv 2>&1
