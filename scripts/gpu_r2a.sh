#!/bin/bash
# round-2 iteration: new parity tests + DP layer groups A/B on the bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dp.py tests/test_gpu_e2e.py tests/test_gpu_qsgd.py tests/test_gpu_psgd.py tests/test_gpu_ddp.py tests/test_gpu_c5.py -m gpu -q -x ${PYTEST_K} > gpurun_out/pytest_r2a.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r2a.log
for g in 1 2; do
  LGRECO_DP_GROUPS=$g timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/bench_g$g.log 2>&1
done
echo done
