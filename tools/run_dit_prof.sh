#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python tools/time_add_norm.py > gpurun_out/add_norm.log 2>&1
