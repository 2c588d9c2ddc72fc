#!/bin/bash
# Short gpurun iteration: selected GPU tests, a no-extras bench, optional ncu capture
# of one kernel (NCU_K=regex).  Usage: TESTS="tests/test_gpu_qsgd.py" NCU_K=k_qprofile bash scripts/gpu_iter.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
[ -f paper_2210_17357_b200/liblgreco.so ] || make all > gpurun_out/make.log 2>&1
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest $TESTS -m gpu -q -x > gpurun_out/pytest_iter.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_iter.log
fi
timeout 600 python bench.py --steps ${BENCH_STEPS:-30} --warmup 5 --no-cpu-baseline --no-extras ${BENCH_ARGS} > gpurun_out/bench_iter.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_iter.log
if [ -n "$NCU_K" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -s ${NCU_S:-2} -c 1 \
    -o gpurun_out/prof_iter -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras ${BENCH_ARGS} > gpurun_out/ncu_iter.log 2>&1
fi
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > gpurun_out/extra.log 2>&1; fi
echo done
