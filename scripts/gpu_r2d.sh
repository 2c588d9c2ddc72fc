#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_ddp.py tests/test_gpu_time_weights.py tests/test_gpu_qsgd.py -m gpu -q > gpurun_out/pytest_d.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_d.log
for v in 2 1; do
  LGRECO_DP_GROUPS=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-extras 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('groups=$v', 'step', d['ms_per_step'], 'kernel', d['roofline']['kernel_ms'], 'pipe', d.get('pipelined_stage_ms'), 'same', d['same_step']['stage_ms'])" >> gpurun_out/ab_groups.log
done
echo done
