#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python tools/time_pinned_e2e.py > gpurun_out/pinned.log 2>&1
