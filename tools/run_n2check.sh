#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
TB_BENCH_GLOO_CHECK=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --no-fp8 --no-configs --no-cpu-baseline --no-w8a8 --dit-layers 2 --dit-samples 1 > gpurun_out/n2check.log 2>&1; echo "rc=$?" >> gpurun_out/n2check.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_arm.log 2>&1; echo "rc=$?" >> gpurun_out/ref_arm.log
