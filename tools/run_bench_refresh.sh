#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
