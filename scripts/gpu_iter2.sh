#!/bin/bash
# targeted GPU tests (PYTEST_FILES) + bench (BENCH_ARGS) + optional ncu of the fused kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest ${PYTEST_FILES} -m gpu -q > gpurun_out/pytest_iter.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_iter.log
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench_iter.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_iter.log
if [ -n "$NCU_FUSED" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_qprofile_q -c 2 -s 3 \
    -o gpurun_out/fused_full -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_fused.log 2>&1
  echo "ncu exit $?" >> gpurun_out/ncu_fused.log
fi
if [ -n "$LAUNCHES" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_iter.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1
fi
echo done
