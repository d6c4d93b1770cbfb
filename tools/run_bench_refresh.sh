#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/step_timeline.py 3 > gpurun_out/timeline.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_sla_step.csv \
    python bench.py --steps 2 --warmup 3 --no-dit --no-fp8 --no-w8a8 --no-configs --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
