#!/bin/bash
# ncu captures of round 2 (run on the GPU box via gpurun; never multi-rank)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
# 1. fused attention kernel at cfg4 (one launch, the bench's timed build)
ncu --set full --clock-control none --import-source on -k regex:sla_tc_kernel -s 3 -c 1 \
    -o gpurun_out/r02_sla_tc_full -f python tools/time_sla.py > gpurun_out/ncu_sla.log 2>&1
ncu -i gpurun_out/r02_sla_tc_full.ncu-rep --page raw --csv > gpurun_out/r02_sla_tc_raw.csv 2>&1
# 2. launch list of the bench steps (every kernel with its device time)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_sla_step.csv \
    python bench.py --steps 2 --warmup 3 --no-dit --no-fp8 --no-w8a8 --no-configs --no-cpu-baseline \
    > gpurun_out/ncu_launch.log 2>&1
