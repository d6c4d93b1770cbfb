#!/bin/bash
# ncu source-level capture of the cfg4 top-k kernel (one launch)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:topk16 -s 1 -c 1 -o gpurun_out/topk_full -f \
    python tools/time_topk.py > gpurun_out/ncu_topk.log 2>&1
ncu -i gpurun_out/topk_full.ncu-rep --page source --csv --print-source sass > gpurun_out/topk_source.csv 2>&1
ncu -i gpurun_out/topk_full.ncu-rep --page raw --csv > gpurun_out/topk_raw.csv 2>&1
