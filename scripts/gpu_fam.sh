#!/bin/bash
# Family baselines: timings + launch lists + ncu captures (exported to CSV on the box, the
# .ncu-rep removed so gpurun_out stays small) on the recipe inputs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
[ -f paper_2210_17357_b200/liblgreco.so ] || make all > gpurun_out/make.log 2>&1
for c in ${FAMS:-C2 C3}; do
  timeout 300 python scripts/family_prof.py $c 5 > gpurun_out/fam_$c.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fam_$c.csv \
    python scripts/family_prof.py $c 2 > /dev/null 2>&1
  if [ -n "$NCU_FULL" ]; then
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_}" -s ${NCU_S:-0} -c ${NCU_C:-30} \
      -o /tmp/prof_fam_$c -f python scripts/family_prof.py $c 2 > gpurun_out/ncu_fam_$c.log 2>&1
    ncu -i /tmp/prof_fam_$c.ncu-rep --page raw --csv > gpurun_out/prof_fam_${c}_raw.csv 2>/dev/null
    python scripts/ncu_summary.py /tmp/prof_fam_$c.ncu-rep gpurun_out/prof_fam_${c}_sum >> gpurun_out/ncu_fam_$c.log 2>&1
  fi
done
echo done
