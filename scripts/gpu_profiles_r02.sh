#!/bin/bash
# Round-2 ncu evidence (never a bench value): the C4 headline launch list + one full
# capture of its kernels, PowerSGD (C2 full capture incl. tensor-pipe counters, C5 launch
# list) and TopK (C3 full capture + launch list).  Summaries via scripts/ncu_summary.py.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/r02
O=gpurun_out/r02
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_qprofile_q|k_qpack|k_solve_cl|k_qprofile_reduce" -s 8 -c 4 \
  -o /tmp/r02_c4 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > $O/ncu_c4.log 2>&1
python scripts/ncu_summary.py /tmp/r02_c4.ncu-rep $O/r02_c4_full $O/launches_c4.csv >> $O/ncu_c4.log 2>&1
ncu -i /tmp/r02_c4.ncu-rep --page raw --csv > $O/r02_c4_raw.csv 2>/dev/null
for c in C2 C3; do
  timeout 900 ncu --set full --clock-control none -k regex:"k_ps_|k_tk_" -s ${S:-30} -c 40 \
    -o /tmp/r02_$c -f python scripts/family_prof.py $c 3 > $O/ncu_$c.log 2>&1
  python scripts/ncu_summary.py /tmp/r02_$c.ncu-rep $O/r02_${c}_full >> $O/ncu_$c.log 2>&1
done
for c in C2 C3 C5p C5t; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
    python scripts/family_prof.py $c 2 > /dev/null 2>&1
done
echo done
