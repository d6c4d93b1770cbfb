#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/profile_dit_block.py > gpurun_out/dit_block.log 2>&1
