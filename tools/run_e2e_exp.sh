#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_capi.py -x -q -k "host" > gpurun_out/e2e_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/e2e_tests.log
timeout 300 python tools/time_host_stage.py > gpurun_out/host_stage.log 2>&1
E2E_CHUNKS=1,2,4 timeout 900 python tools/time_dropin_e2e.py > gpurun_out/e2e_dropin.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
