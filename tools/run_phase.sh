#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
TB200_LIB=$PWD/paper_2512_16093_b200/libtb200_trace.so timeout 300 python tools/trace_sla.py > gpurun_out/trace.log 2>&1
