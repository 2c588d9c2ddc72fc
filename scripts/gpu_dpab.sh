#!/bin/bash
# DP solve configuration A/B in the pipelined schedule (groups x cluster size)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for cfg in "2 16" "1 16" "1 8" "2 8" "1 4"; do
  set -- $cfg
  LGRECO_DP_GROUPS=$1 LGRECO_DP_NC=$2 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-extras 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('groups=$1 nc=$2', 'step', d['ms_per_step'], 'kernel', d['roofline']['kernel_ms'], 'pipe', d.get('pipelined_stage_ms'), 'same', d['same_step']['stage_ms'])" >> gpurun_out/ab_dp.log
done
echo done
