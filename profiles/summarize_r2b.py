"""Round-3 ncu summary: the --set full captures of profiles/r2b_final_b.sh (g_*_raw.csv, g_*_hot_lines.txt,
exported on the box) and the launch list of profiles/r2b_final_a.sh, as markdown.

    python profiles/summarize_r2b.py --dir gpurun_out --out profiles/r2b_cfg3_ncu.md
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_raw import METRICS, launch_table, read_raw  # noqa: E402

CAPS = [
    ("g_count", "cfg3 radius count, r = 1 (`radius_pt_kernel`, point prefilter, coarse 256)"),
    ("g_fill", "cfg3 radius fill (row-major replay), r = 1"),
    ("g_sort", "cfg3 onesweep pass (one of 8; pipelined ranking, 4-wide look-back)"),
    ("g_gather", "cfg3 gather into SFC order (4 record gathers in flight per thread)"),
    ("g_c1_count_r3", "cfg1 radius count, r = 3"),
    ("g_c1_sort", "cfg1 onesweep pass (one of 8)"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", default="gpurun_out")
    ap.add_argument("--out", default="profiles/r2b_cfg3_ncu.md")
    ap.add_argument("--launches", default="profiles/r2b/launches_cfg3.csv")
    a = ap.parse_args()
    L = ["# ncu summary -- round 2, second session (cfg3, plus cfg1 count at r = 3 and a cfg1 sort pass)", "",
         "One B200. `--set full --clock-control none --import-source on` captures by `profiles/r2b_final_b.sh`, "
         "each after the same command exited 0 without ncu; launch list by `profiles/r2b_final_a.sh`. ncu times "
         "are cold-cache and serialised: compare shares, not absolute times, with the bench line.", ""]
    agg = launch_table(a.launches)
    tot = sum(v[1] for v in agg.values()) or 1.0
    L += ["## Launch list (`bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-knn --no-extra`)", "",
          "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        L.append(f"| `{k}` | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")
    L.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.3f} | 100% |")
    for name, desc in CAPS:
        raw = os.path.join(a.dir, f"{name}_raw.csv")
        if not os.path.exists(raw):
            continue
        recs = read_raw(raw)
        if not recs:
            continue
        r = recs[0]
        L += ["", f"## {desc} (`{name}`)", "", f"| metric | `{r['kernel']}` |", "|---|---|"]
        for m in METRICS:
            if m in r:
                v = r[m]
                if m.startswith("dram__bytes"):
                    L.append(f"| {m} | {v / 1e9:.3f} GB |")
                elif m == "gpu__time_duration.sum":
                    L.append(f"| {m} | {v:.3f} ms |")
                else:
                    L.append(f"| {m} | {v:.2f} |")
        hot = os.path.join(a.dir, f"{name}_hot_lines.txt")
        if os.path.exists(hot):
            L += ["", "Hottest source lines (share of warp samples, share of instructions, threads per instruction):",
                  "", "```"] + open(hot).read().splitlines()[:16] + ["```"]
    open(a.out, "w").write("\n".join(L) + "\n")
    print(a.out)


if __name__ == "__main__":
    main()
