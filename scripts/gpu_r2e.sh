#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_dp.py -m gpu -q > gpurun_out/pytest_e.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_e.log
timeout 900 python bench.py > gpurun_out/bench_e.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_e.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_e.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1
echo done
