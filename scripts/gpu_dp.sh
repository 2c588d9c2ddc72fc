#!/bin/bash
# DP iteration: phase timing (C4), DP parity tests, a short headline bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
DP_ONLY_C4=1 timeout 200 python scripts/dp_timing.py timing > gpurun_out/dpt.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dp.py tests/test_gpu_e2e.py ${DP_TESTS} -q -x -m gpu > gpurun_out/pt_dp.log 2>&1; echo "pytest exit $?" >> gpurun_out/pt_dp.log
timeout 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/bench.log 2>&1
tail -2 gpurun_out/pt_dp.log; grep -o "\"ms_per_step\": [0-9.]*\|\"solve\": [0-9.]*" gpurun_out/bench.log | head -2
