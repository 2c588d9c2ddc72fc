#!/usr/bin/env python
"""Summarise an ncu --set full report (and optionally a launch-list CSV) into a
markdown table + JSON under profiles/.  Usage:
  python scripts/ncu_summary.py gpurun_out/prof_full.ncu-rep profiles/r01_full [gpurun_out/launches.csv]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "time_us": ("gpu__time_duration.sum", 1e-3),  # ns -> us
    "dram_read_MB": ("dram__bytes_read.sum", None),
    "dram_write_MB": ("dram__bytes_write.sum", None),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "inst_executed": ("smsp__inst_executed.sum", 1),
    "registers": ("launch__registers_per_thread", 1),
    "tensor_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "fp64_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "fma_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
}
STALLS = ["long_scoreboard", "wait", "math_pipe_throttle", "short_scoreboard", "barrier", "mio_throttle",
          "lg_throttle", "not_selected", "selected", "dispatch_stall", "no_instructions"]


def _to_mb(v, unit):
    v = float(v)
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
    return v * scale


def _f(v):
    try:
        return f"{float(v):.1f}"
    except (TypeError, ValueError):
        return "-"


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in rows[2:]:
        d = {"kernel": r[col["Kernel Name"]].split("(")[0]}
        for k, (m, sc) in METRICS.items():
            if m not in col:
                continue
            v, u = r[col[m]], units[col[m]]
            try:
                if k.endswith("_MB"):
                    d[k] = round(_to_mb(v.replace(",", ""), u), 3)
                elif k == "time_us":
                    fv = float(v.replace(",", ""))
                    d[k] = round(fv * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1e-3), 3)
                else:
                    d[k] = float(v.replace(",", ""))
            except ValueError:
                d[k] = v
        st = {}
        for s in STALLS:
            m = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if m in col:
                try:
                    st[s] = int(float(r[col[m]].replace(",", "")))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1
        d["top_stalls"] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda x: -x[1])[:4]}
        res.append(d)
    json.dump(res, open(out + ".json", "w"), indent=1)
    with open(out + ".md", "w") as f:
        f.write(f"ncu --set full summary of `{rep}`\n\n")
        f.write("| kernel | us | DRAM R MB | DRAM W MB | DRAM % | issue % | warps % | tensor % | fp64 % | inst | regs | "
                "top stalls |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|---|---|\n")
        for d in res:
            f.write(f"| {d['kernel']} | {d.get('time_us')} | {d.get('dram_read_MB')} | {d.get('dram_write_MB')} | "
                    f"{d.get('dram_pct', 0):.1f} | {d.get('issue_active_pct', 0):.1f} | {d.get('warps_active_pct', 0):.1f} | "
                    f"{_f(d.get('tensor_pct'))} | {_f(d.get('fp64_pct'))} | "
                    f"{int(d.get('inst_executed', 0))} | {int(d.get('registers', 0))} | "
                    f"{', '.join(f'{k} {v}' for k, v in d['top_stalls'].items())} |\n")
    if len(sys.argv) > 3:  # launch list -> per-kernel share of device time
        lines = open(sys.argv[3]).read().splitlines()
        start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
        tot, ours, per, cnt = 0.0, 0.0, {}, {}
        for r in csv.DictReader(io.StringIO("\n".join(lines[start:]))):
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = r["Kernel Name"].split("(")[0]
            v = float(r["Metric Value"].replace(",", ""))
            per[name] = per.get(name, 0.0) + v
            cnt[name] = cnt.get(name, 0) + 1
            tot += v
            if "lg::" in name:
                ours += v
        with open(out + "_launches.md", "w") as f:
            f.write("Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised: "
                    "compare shares, not absolutes).  `share` = of all device time in the list; `share_lg` = of the "
                    "library's own kernels (lg::*), i.e. of the hot path without the bench's L2-flush memsets and "
                    "input fills.\n\n| kernel | launches | total us | mean us | share | share_lg |\n|---|---|---|---|---|---|\n")
            for k, v in sorted(per.items(), key=lambda x: -x[1]):
                sl = f"{v / ours:.3f}" if "lg::" in k and ours else "-"
                f.write(f"| {k} | {cnt[k]} | {v / 1e3:.1f} | {v / 1e3 / cnt[k]:.1f} | {v / tot:.3f} | {sl} |\n")


if __name__ == "__main__":
    main()
