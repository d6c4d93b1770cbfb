#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
: > gpurun_out/e2e_threads.log
for r in 1 2; do
for t in 16 14 12; do
  echo "threads $t" >> gpurun_out/e2e_threads.log
  TB_HOST_THREADS=$t E2E_MODES="bf16-valued;f32-valued" E2E_CHUNKS=4 timeout 600 python tools/time_dropin_e2e.py 2>&1 | cut -c1-110 >> gpurun_out/e2e_threads.log
done; done
