#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for g in 1 2; do
  LGRECO_DP_GROUPS=$g DP_ONLY_C4=1 timeout 300 python scripts/dp_timing.py timing > gpurun_out/dpt_g$g.log 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_ddp.py tests/test_gpu_c5.py -m gpu -q -x > gpurun_out/pytest_r2b.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r2b.log
echo done
