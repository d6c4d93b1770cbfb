#!/bin/bash
# ncu source-level capture of the fast 2-SM W8A8 kernel at the DiT qkv shape (one launch)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:w8a8_2sm -s 1 -c 1 \
    -o gpurun_out/w8_full -f python tools/gemm_one.py 75600 5120 15360 0 1 > gpurun_out/ncu_w8.log 2>&1
ncu -i gpurun_out/w8_full.ncu-rep --page source --csv --print-source sass > gpurun_out/w8_source.csv 2>&1
ncu -i gpurun_out/w8_full.ncu-rep --page raw --csv > gpurun_out/w8_raw.csv 2>&1
ls -la gpurun_out
