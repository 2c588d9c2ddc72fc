# A/B of library variants built by scripts/build_variants.sh (LGRECO_LIB); results -> gpurun_out/ab.log
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then unset LGRECO_LIB; else export LGRECO_LIB=$PWD/build/var/liblgreco_$v.so; fi
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-extras ${AB_ARGS} 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'step', d['ms_per_step'], 'kernel', d['roofline']['kernel_ms'], 'pipe', d.get('pipelined_stage_ms'), 'same', d['same_step']['stage_ms'])" >> gpurun_out/ab.log
done
done
