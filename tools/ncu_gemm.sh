#!/bin/bash
# ncu capture of the coverage GEMM (tb_gemm_bf16_batched) at cfg4, one launch
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -c 1 -o gpurun_out/gemm_full -f \
    python tools/time_sla.py > gpurun_out/ncu_gemm.log 2>&1
ncu -i gpurun_out/gemm_full.ncu-rep --page raw --csv > gpurun_out/gemm_raw.csv 2>&1
ncu -i gpurun_out/gemm_full.ncu-rep --page source --csv --print-source sass > gpurun_out/gemm_source.csv 2>&1
