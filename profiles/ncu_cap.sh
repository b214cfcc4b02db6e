#!/bin/bash
# sourced: cap NAME KERNEL_REGEX "EXTRA_NCU_ARGS" COMMAND... -> gpurun_out/NAME_raw.csv, NAME_hot_lines.txt
NCU="ncu --set full --clock-control none --import-source on"
cap() {
  local name=$1 re=$2 extra=$3; shift 3
  timeout 900 $NCU -f -k regex:"$re" $extra -o /tmp/$name "$@" > gpurun_out/ncu_$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${name}_src.csv 2>/dev/null
  python - "$name" <<'PY'
import csv, sys
name = sys.argv[1]
rows = list(csv.reader(open(f"/tmp/{name}_src.csv")))
cur, out = None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if len(r) > 8 and r[0].isdigit() and r[2] == '-':
        try: out.append((int(r[4]), int(r[7]), int(r[8]), cur, int(r[0]), r[1][:110]))
        except ValueError: pass
ts = sum(o[0] for o in out) or 1; ti = sum(o[1] for o in out) or 1
with open(f"gpurun_out/{name}_hot_lines.txt", "w") as f:
    f.write("samples% inst% threads/inst  file:line  source\n")
    for o in sorted(out, key=lambda o: -o[0])[:40]:
        f.write(f"{100*o[0]/ts:6.1f} {100*o[1]/ti:6.1f} {o[2]/max(o[1],1):5.1f}  {o[3]}:{o[4]}  {o[5]}\n")
PY
}
