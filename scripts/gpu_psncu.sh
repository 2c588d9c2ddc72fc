#!/bin/bash
# ncu --set full of the PowerSGD kernels on a family config (C2 default): the tensor
# pipe / fp64 pipe / DRAM counters for profiles/r02_psgd.md
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
c=${FAM:-C2}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_ps_}" -s ${NCU_S:-40} -c ${NCU_C:-40} \
  -o /tmp/prof_ps_$c -f python scripts/family_prof.py $c 3 > gpurun_out/ncu_ps_$c.log 2>&1
python scripts/ncu_summary.py /tmp/prof_ps_$c.ncu-rep gpurun_out/prof_ps_${c}_sum >> gpurun_out/ncu_ps_$c.log 2>&1
ncu -i /tmp/prof_ps_$c.ncu-rep --page raw --csv > gpurun_out/prof_ps_${c}_raw.csv 2>/dev/null
echo done
