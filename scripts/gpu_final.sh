#!/bin/bash
# round-end style check: full GPU suite, smoke, default bench, launch list of the pipelined step
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_final.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_final.log
LG_MULTI_ONE_DEVICE=1 timeout 600 python -m pytest tests/test_gpu_multigpu.py -m gpu -q -k p2p > gpurun_out/multi_onedev.log 2>&1; echo "exit $?" >> gpurun_out/multi_onedev.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1
echo done
