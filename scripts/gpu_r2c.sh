#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_all.log
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_full.log
for v in 0 1; do
  LGRECO_K1B=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-extras 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('K1B=$v', 'step', d['ms_per_step'], 'kernel', d['roofline']['kernel_ms'], 'pipe', d.get('pipelined_stage_ms'), 'same', d['same_step']['stage_ms'])" >> gpurun_out/ab_k1b.log
done
echo done
