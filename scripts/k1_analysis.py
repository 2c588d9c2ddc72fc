#!/usr/bin/env python
"""Summarise an ncu source-level capture of K1 (k_qprofile_q) into markdown: warp
instructions per element, the SASS mix of the hot loop, pipe utilisation and the stall
breakdown.  Inputs are the CSV exports of one `ncu --set full --import-source on`
report (`--page source --csv --print-source sass` and `--page raw --csv`).  Usage:
  python scripts/k1_analysis.py gpurun_out/k1_sass.csv gpurun_out/k1_raw.csv N_ELEMENTS > profiles/r01_k1_analysis.md
"""
import collections
import csv
import sys


def main():
    sass_csv, raw_csv, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
    rows = list(csv.reader(open(sass_csv)))
    hdr = rows[1]
    data = rows[2:]
    ia = hdr.index("Instructions Executed")
    isrc = hdr.index("Source")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[ia]) for r in data)
    mix = collections.Counter()
    for r in data:
        op = r[isrc].strip().split()
        if not op:
            continue
        k = op[0]
        if k.startswith("@"):
            k = op[1] if len(op) > 1 else k
        mix[k.split(".")[0]] += int(r[ia])
    raw = list(csv.reader(open(raw_csv)))
    h, v = raw[0], raw[2]

    def m(name):
        return float(v[h.index(name)]) if name in h else float("nan")

    print("# K1 (`k_qprofile_q<7>`, C4) source-level ncu summary\n")
    print(f"Elements: {n:,}.  Kernel time under ncu: {m('gpu__time_duration.sum'):.1f} us (cold, serialised).\n")
    print(f"Warp instructions executed: {tot:,} = **{32 * tot / n:.1f} lane-instructions per element**.\n")
    print("| pipe / metric | % of peak (active) |")
    print("|---|---|")
    for name, label in [("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active"),
                        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe"),
                        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe"),
                        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe"),
                        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe"),
                        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (occupancy)"),
                        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput")]:
        print(f"| {label} | {m(name):.1f} |")
    print("\nSASS mix (executed warp instructions, top 16; per element = x32/N):\n")
    print("| opcode | warp instr | per element |")
    print("|---|---|---|")
    for k, c in mix.most_common(16):
        print(f"| {k} | {c:,} | {32 * c / n:.2f} |")
    stalls = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: float(v[h.index(k)]) for k in h
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
    st = sum(stalls.values())
    print("\nWarp-state samples (all):\n")
    print("| reason | share |")
    print("|---|---|")
    for k, c in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]:
        print(f"| {k} | {c / st:.3f} |")


if __name__ == "__main__":
    main()
