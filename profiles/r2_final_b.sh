#!/bin/bash
# Round 2 evidence pass B: --set full captures of the top kernels (after the plain run exited 0);
# exported on the box as raw-metric and source-level CSV (the reports stay under the 64 MiB limit
# only for the headline kernel).
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
P="python profiles/run_profile.py --config cfg3 --reps 1"
timeout 600 $P --radius 1.0 --k 16 --fingerprint > $OUT/final_prof.log 2>&1 || exit 1
NCU="ncu --set full --clock-control none --import-source on"
cap() {  # name, kernel regex, extra ncu args, command...
  local name=$1 re=$2 extra=$3; shift 3
  timeout 900 $NCU -k regex:"$re" $extra -o /tmp/$name "$@" > $OUT/ncu_$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
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
cap f_count radius_pt_kernel "-c 1" $P --radius 1.0
cp /tmp/f_count.ncu-rep $OUT/
cap f_fill radius_replay "-c 1" $P --radius 1.0
cap f_digest radius_digest "-c 1" $P --radius 1.0 --fingerprint
cap f_sort onesweep_pass "-s 3 -c 1" $P --radius
cap f_reorder "gather_soa|encode_kernel|bbox_kernel" "-c 3" $P --radius
cap f_build "open_count|open_emit|link_nodes|emit_tnodes|tnode" "-c 7" $P --radius
cap f_knn16 knn_float_kernel "-c 1" $P --radius --k 16
cap f_c1_knn64 knn_float_kernel "-c 1" python profiles/run_profile.py --config cfg1 --reps 1 --radius --k 64
cap f_c1_count_r3 radius_pt_kernel "-s 3 -c 1" python profiles/run_profile.py --config cfg1 --reps 1 --radius 0.5 1.0 2.0 3.0
du -sh $OUT; ls -la $OUT
exit 0
