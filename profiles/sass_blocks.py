"""Per-basic-block instruction / stall-sample shares of one kernel in an ncu report (read here,
no GPU):  python profiles/sass_blocks.py report.ncu-rep [kernel-regex] [min-share]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else None
    thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if kre:
        cmd += ["-k", f"regex:{kre}"]
    rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
    seen, ins = set(), []
    for r in rows:
        if len(r) < 6 or r[0] == "Address":
            continue
        try:
            a, n, smp = int(r[0], 16), int(r[5]), int(r[2])
        except ValueError:
            continue
        if a in seen:
            continue
        seen.add(a)
        ins.append((a, r[1].strip(), n, smp))
    ins.sort()
    blocks, cur = [], None
    for a, s, n, smp in ins:
        if cur and cur["n"] == n:
            cur["end"] = a
            cur["len"] += 1
            cur["smp"] += smp
            cur["top"].append((smp, s))
        else:
            cur = {"start": a, "end": a, "n": n, "len": 1, "smp": smp, "top": [(smp, s)]}
            blocks.append(cur)
    ti = sum(b["n"] * b["len"] for b in blocks) or 1
    ts = sum(b["smp"] for b in blocks) or 1
    print(f"instructions {ti:.3e}  samples {ts}")
    for b in blocks:
        fi, fs = b["n"] * b["len"] / ti, b["smp"] / ts
        if fi >= thr or fs >= thr:
            top = [t[1][:34] for t in sorted(b["top"], reverse=True)[:3]]
            print(f"{b['start'] & 0xfffff:05x}-{b['end'] & 0xfffff:05x} x{b['n']:>11} len {b['len']:3d} "
                  f"inst {100 * fi:5.1f}% smp {100 * fs:5.1f}%  {top}")


if __name__ == "__main__":
    main()
