"""Summarise ncu `--page raw --csv` exports (one file per capture, written on the GPU box by
profiles/r2_final_b.sh) into a markdown report and profiles/traffic.json.

    python profiles/summarize_raw.py --dir gpurun_out --out profiles/r2_cfg3_ncu.md \\
        --launches profiles/r2/launches_cfg3.csv --traffic profiles/traffic.json
"""
import argparse
import collections
import csv
import json
import os

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "launch__registers_per_thread",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]
SCALE = {"ms": 1.0, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6, "msecond": 1.0, "s": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

# capture -> (description, bench stage it measures, config)
CAPTURES = {
    "f_count": ("cfg3 radius count, r = 1", "radius_count@r=1.0"),
    "f_fill": ("cfg3 radius fill (replay), r = 1", "radius_fill@r=1.0"),
    "f_digest": ("cfg3 FNV-1a row digests, r = 1", "radius_digest@r=1.0"),
    "f_scan": ("cfg3 u64 scan of the counts, r = 1", "radius_scan@r=1.0"),
    "f_sort": ("cfg3 onesweep pass (one of 8)", "sort"),
    "f_reorder": ("cfg3 bbox / encode / gather", None),
    "f_build": ("cfg3 octree build kernels", None),
    "f_knn16": ("cfg3 kNN k = 16", None),
    "f_c1_knn64": ("cfg1 kNN k = 64", None),
    "f_c1_count_r3": ("cfg1 radius count, r = 3", None),
}


def read_raw(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        rec = {"kernel": r[col["Kernel Name"]].split("(")[0]}
        for m in METRICS:
            i = col.get(m)
            if i is None or r[i] in ("", "n/a"):
                continue
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if m == "gpu__time_duration.sum":
                v *= SCALE.get(u, 1.0)  # -> ms
            elif m.startswith("dram__bytes"):
                v *= SCALE.get(u, 1.0)  # -> bytes
            rec[m] = v
        out.append(rec)
    return out


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3}.get(d["Metric Unit"], 1.0)
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    return agg


def stage_traffic(path):
    """Per-stage DRAM bytes from a per-launch ncu list of one step (kernels in launch order)."""
    rows = list(csv.reader(open(path)))
    hdr = None
    launches = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        rec = launches.setdefault(int(d["ID"]), {"kernel": d["Kernel Name"].split("(")[0]})
        v = float(d["Metric Value"].replace(",", ""))
        v *= SCALE.get(d["Metric Unit"], 1.0)
        if d["Metric Name"] == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", "")) * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3,
                                                              "usecond": 1e-3}.get(d["Metric Unit"], 1.0)
        rec[d["Metric Name"]] = v
    stages = collections.OrderedDict()
    phase = "reorder"
    for _, rec in sorted(launches.items()):
        k = rec["kernel"]
        if "radius_pt_kernel" in k:
            phase, st = "scan", "radius_count"
        elif "radius_replay" in k:
            phase, st = "fill", "radius_fill"
        elif "radius_digest" in k:
            st = "radius_digest"
        elif phase == "scan":
            st = "radius_scan"
        elif "bbox" in k:
            st = "bbox"
        elif "encode_kernel" in k:
            st = "encode"
        elif "onesweep" in k or "sort_bases" in k or "iota" in k:
            st = "sort"
        elif "gather_soa" in k:
            st = "gather"
        elif k in ("tnode_float", "float_points"):
            st = "float_shadows"
        elif phase == "reorder" and k.startswith("fetch_words"):
            continue
        else:
            st = "build"
        agg = stages.setdefault(st, {"dram": 0.0, "ms": 0.0, "kernels": collections.Counter()})
        agg["dram"] += rec.get("dram__bytes_read.sum", 0.0) + rec.get("dram__bytes_write.sum", 0.0)
        agg["ms"] += rec.get("gpu__time_duration.sum", 0.0)
        agg["kernels"][k] += 1
    return stages


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", default="gpurun_out")
    ap.add_argument("--out", default="profiles/r2_cfg3_ncu.md")
    ap.add_argument("--launches", default="profiles/r2/launches_cfg3.csv")
    ap.add_argument("--traffic", default="profiles/traffic.json")
    ap.add_argument("--traffic-launches", default="profiles/r2/traffic_launches_cfg3.csv",
                    help="per-launch DRAM bytes of one step (every kernel)")
    a = ap.parse_args()
    md = ["# ncu summary — round 2 final code (cfg3, plus cfg1 kNN k = 64 and count r = 3)", "",
          "One B200. Captures: `profiles/r2_final_b.sh` (`ncu --set full --clock-control none --import-source on`, "
          "exported on the box with `--page raw --csv` and `--page source --csv`); launch list: "
          "`profiles/r2_final_a.sh`. Every capture ran after the same command exited 0 without ncu. ncu times "
          "are cold-cache and serialised, so compare shares, not absolute times, with the bench line.", ""]
    if os.path.exists(a.launches):
        agg = launch_table(a.launches)
        tot = sum(v[1] for v in agg.values())
        md += ["## Launch list (`--metrics gpu__time_duration.sum --clock-control none`, "
               "`bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-knn --no-extra`)", "",
               "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            md.append(f"| `{k}` | {v[0]} | {v[1]:.3f} | {100 * v[1] / tot:.1f}% |")
        md += [f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.3f} | 100% |", ""]
    traffic = {"config": "cfg3", "stages": {}}
    for cap, (desc, stage) in CAPTURES.items():
        path = os.path.join(a.dir, f"{cap}_raw.csv")
        if not os.path.exists(path):
            continue
        recs = read_raw(path)
        if not recs:
            continue
        md += [f"## {desc} (`{cap}`)", ""]
        names = [r["kernel"] for r in recs]
        md += ["| metric | " + " | ".join(f"`{n}`" for n in names) + " |",
               "|---|" + "---|" * len(recs)]
        for m in METRICS:
            vals = []
            for r in recs:
                v = r.get(m)
                if v is None:
                    vals.append("")
                elif m == "gpu__time_duration.sum":
                    vals.append(f"{v:.3f} ms")
                elif m.startswith("dram__bytes"):
                    vals.append(f"{v / 1e9:.3f} GB")
                else:
                    vals.append(f"{v:.2f}")
            md.append(f"| {m} | " + " | ".join(vals) + " |")
        md.append("")
        hot = os.path.join(a.dir, f"{cap}_hot_lines.txt")
        if os.path.exists(hot):
            lines = open(hot).read().splitlines()[:16]
            md += ["Hottest source lines (share of warp samples, share of instructions, threads per instruction):",
                   "", "```"] + lines + ["```", ""]
        if stage:
            r = recs[0]
            traffic["stages"][stage] = {
                "dram_bytes_per_launch": r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0),
                "issue_active_pct": r.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "warps_active_pct": r.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
                "l2_hit_pct": r.get("lts__t_sector_hit_rate.pct"),
                "kernel": r["kernel"],
                "ncu_ms": r.get("gpu__time_duration.sum"),
                "source": f"{os.path.basename(a.out)} ({cap}, ncu --set full)",
            }
    open(a.out, "w").write("\n".join(md) + "\n")
    if os.path.exists(a.traffic_launches):
        st = stage_traffic(a.traffic_launches)
        md += ["## DRAM traffic per stage (one cfg3 step, r = 1; `ncu --metrics dram__bytes_read.sum,"
               "dram__bytes_write.sum,gpu__time_duration.sum` over every kernel, cold-cache and serialised)", "",
               "| stage | kernels | DRAM GB | ncu ms |", "|---|---|---|---|"]
        for name, agg in st.items():
            ks = ", ".join(f"`{k}` x{c}" for k, c in agg["kernels"].items())
            md.append(f"| {name} | {ks} | {agg['dram'] / 1e9:.3f} | {agg['ms']:.3f} |")
            key = name + "@r=1.0" if name.startswith("radius_") else name
            full = traffic["stages"].get(key, {})
            traffic["stages"][key] = {
                "dram_bytes_per_launch": agg["dram"],
                "issue_active_pct": full.get("issue_active_pct"),
                "warps_active_pct": full.get("warps_active_pct"),
                "l2_hit_pct": full.get("l2_hit_pct"),
                "kernel": " + ".join(agg["kernels"]),
                "source": f"{os.path.basename(a.traffic_launches)} (every kernel of the stage, one step)"
                          + (f"; issue from {full['source']}" if full.get("source") else ""),
            }
        md.append("")
        open(a.out, "w").write("\n".join(md) + "\n")
    if traffic["stages"]:
        json.dump(traffic, open(a.traffic, "w"), indent=1)
    print(f"wrote {a.out} ({len(md)} lines), traffic stages: {sorted(traffic['stages'])}")


if __name__ == "__main__":
    main()
