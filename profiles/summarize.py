"""Summarise ncu outputs (read here, no GPU) into profiles/<tag>_*.md and profiles/traffic.json.

    python profiles/summarize.py --tag r1 --launches gpurun_out/launches.csv \
        --rep gpurun_out/fill.ncu-rep --stage "radius_fill@r=3.0" --config cfg1
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
]


def launches_table(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg: dict[str, list] = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
        a = agg.setdefault(name, [0.0, 0])
        a[0] += v * scale
        a[1] += 1
    tot = sum(v[0] for v in agg.values())
    out = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for name, (ms, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        out.append(f"| `{name}` | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")
    out.append(f"| **total** | {sum(v[1] for v in agg.values())} | {tot:.3f} | 100% |")
    return "\n".join(out)


def raw_metrics(rep: str) -> list[dict]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = []
    for d in rows[2:]:
        rec = {"kernel": d[h.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in h:
                rec[m] = (d[h.index(m)], units[h.index(m)])
        out.append(rec)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--stage", nargs="*", default=[],
                    help="bench stage names the --rep kernels correspond to (same order)")
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    md = [f"# ncu summary — {a.tag}", ""]
    if a.note:
        md += [a.note, ""]
    if a.launches:
        md += ["## Launch list (`--metrics gpu__time_duration.sum --clock-control none`; cold-cache, "
               "serialised: compare shares)", "", launches_table(a.launches), ""]
    traffic = {}
    for i, rep in enumerate(a.rep):
        recs = raw_metrics(rep)
        for rec in recs:
            md += [f"## `{rec['kernel']}` (`{os.path.basename(rep)}`, --set full)", "",
                   "| metric | value | unit |", "|---|---|---|"]
            for m in METRICS:
                if m in rec:
                    md.append(f"| {m} | {rec[m][0]} | {rec[m][1]} |")
            md.append("")
        if i < len(a.stage) and recs:
            r0 = recs[0]

            def to_bytes(v):
                val, unit = float(v[0].replace(",", "")), v[1]
                return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)

            def pct(m):
                return float(r0[m][0].replace(",", "")) if m in r0 else None
            traffic[a.stage[i]] = {
                "dram_bytes_per_launch": to_bytes(r0["dram__bytes_read.sum"]) + to_bytes(r0["dram__bytes_write.sum"]),
                "issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "warps_active_pct": pct("sm__warps_active.avg.pct_of_peak_sustained_active"),
                "l2_hit_pct": pct("lts__t_sector_hit_rate.pct"),
                "kernel": r0["kernel"],
                "source": f"profiles/{a.tag}_ncu.md ({os.path.basename(rep)}, ncu --set full)"}
    path = os.path.join(HERE, f"{a.tag}_ncu.md")
    open(path, "w").write("\n".join(md) + "\n")
    print("wrote", path)
    if traffic:
        tj = {"config": a.config, "stages": traffic}
        json.dump(tj, open(os.path.join(HERE, "traffic.json"), "w"), indent=1)
        print("traffic", tj)


if __name__ == "__main__":
    main()
