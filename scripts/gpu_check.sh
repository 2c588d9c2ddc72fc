#!/bin/bash
# One gpurun batch: GPU parity tests, smoke, bench, ncu launch list + full capture.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out build
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
[ -f paper_2210_17357_b200/liblgreco.so ] || make all > gpurun_out/make.log 2>&1
timeout 900 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps ${BENCH_STEPS:-50} --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_qprofile_q|k_qpack|k_solve_cl|k_qprofile_reduce" -s 8 -c 4 \
  -o gpurun_out/prof_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_full.log 2>&1
fi
echo done
