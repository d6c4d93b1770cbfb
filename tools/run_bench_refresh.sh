#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 300 python tools/step_timeline.py > gpurun_out/timeline.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1100 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-w8a8 --no-dit --no-configs --no-fp8 > gpurun_out/ncu_launch.log 2>&1
