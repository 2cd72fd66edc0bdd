"""Hot SASS of one kernel from an `ncu --page source --csv --print-source sass` dump:
   python tools/sass_hot.py FILE KERNEL_SUBSTR [occurrence] [top]"""
import csv
import sys

path, want = sys.argv[1], sys.argv[2]
occ = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
blocks, cur = [], None
for r in csv.reader(open(path)):
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        blocks.append(cur)
    elif cur is not None and r and r[0] == "Address":
        cur[1] = {h: i for i, h in enumerate(r)}
    elif cur is not None and cur[1] and r:
        cur[2].append(r)
sel = [b for b in blocks if want in b[0]]
name, ix, rows = sel[occ]
print(name[:120], len(rows), "instructions")
ie, ss = ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"]
tot = sum(float(r[ie] or 0) for r in rows)
tots = sum(float(r[ss] or 0) for r in rows)
print("total warp instr executed", tot, "stall samples", tots)
# per-region listing: print all instructions with their counts in address order, only those >0.5% of max
mx = max(float(r[ie] or 0) for r in rows)
for r in rows:
    e = float(r[ie] or 0)
    s = float(r[ss] or 0)
    if e >= mx * 0.2 or s >= tots * 0.01:
        print(f"{r[ix['Address']]:>6} {e:12.0f} {s:7.0f}  {r[ix['Source']][:90]}")
