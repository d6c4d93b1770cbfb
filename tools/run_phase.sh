#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
TB200_LIB=$PWD/paper_2512_16093_b200/libtb200_trace.so timeout 300 python tools/trace_sla.py > gpurun_out/trace2.log 2>&1
TB_SLA_SMEM_PAD=110000 TB200_LIB=$PWD/paper_2512_16093_b200/libtb200_trace.so timeout 300 python tools/trace_sla.py > gpurun_out/trace1.log 2>&1
