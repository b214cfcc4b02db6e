"""Static SASS evidence, read here (no GPU): per-kernel mnemonic histogram of liblinoct_b200.so
from `cuobjdump -sass`, for the kernels named by regex.

    python profiles/sass_mnemonics.py > profiles/r3/sass_mnemonics.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2603_06771_b200", "liblinoct_b200.so")
KERNELS = [r"radius_pt_kernelILi0ELb0ELi0E", r"radius_replay_kernel", r"radius_digestILb0E", r"onesweep_passILi1E",
           r"gather_soa", r"encode_kernelILi1E", r"knn_float_kernelILb0ELi16ELb0E", r"struct_pt_kernelILi0ELi0E"]
FAMILIES = [("packed f32x2 (FADD2/FMUL2/FFMA2)", r"^(FADD2|FMUL2|FFMA2)"), ("FP32 scalar", r"^(FADD|FMUL|FFMA|FMNMX|FSETP|FSEL)\b"),
            ("FP64", r"^(DADD|DMUL|DFMA|DSETP|F2F)"), ("warp vote / match / shuffle", r"^(VOTE|MATCH|SHFL|REDUX)"),
            ("global loads", r"^(LDG|LD\.)"), ("global stores / atomics", r"^(STG|ST\.|ATOMG|RED\b|RED\.)"),
            ("shared memory", r"^(LDS|STS|ATOMS|LDSM)"), ("local (spills)", r"^(LDL|STL)"),
            ("integer mul-add", r"^(IMAD|IMUL)"), ("branches / barriers", r"^(BRA|BSSY|BSYNC|BAR|WARPSYNC|EXIT)")]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs, cur = {}, None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and cur:
        funcs[cur].append(m.group(1))
print("# SASS mnemonic histogram of the hot kernels (cuobjdump -sass of the in-tree sm_100a build)\n")
print("Static instruction counts, not executed counts; `ncu/*_hot_lines.txt` has the sampled shares.\n")
for kre in KERNELS:
    for name, ins in funcs.items():
        if not re.search(kre, name):
            continue
        fam = collections.Counter()
        for op in ins:
            for label, pat in FAMILIES:
                if re.match(pat, op):
                    fam[label] += 1
                    break
        top = collections.Counter(i.split(".")[0] for i in ins).most_common(8)
        special = sorted({i for i in ins if re.search(r"LTC|\.NC|\.CONSTANT|EF|\.128|\.64\b", i) and i.startswith(("LDG", "STG"))})[:10]
        print(f"## `{name[:70]}`\n\n{len(ins)} instructions. Top: " + ", ".join(f"{o} {c}" for o, c in top) + ".\n")
        print("| family | static count |\n|---|---|")
        for label, _ in FAMILIES:
            print(f"| {label} | {fam[label]} |")
        if special:
            print("\nGlobal access forms: " + ", ".join(f"`{s}`" for s in special))
        print()
        break
