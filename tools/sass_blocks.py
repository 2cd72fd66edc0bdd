"""Basic-block profile of one kernel from an ncu source/SASS CSV: runs of equal
execution count, sorted by warp instructions (count x length).
   python tools/sass_blocks.py FILE KERNEL_SUBSTR [occurrence] [top]"""
import csv
import sys

path, want = sys.argv[1], sys.argv[2]
occ = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
blocks, cur = [], None
for r in csv.reader(open(path)):
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        blocks.append(cur)
    elif cur is not None and r and r[0] == "Address":
        cur[1] = {h: i for i, h in enumerate(r)}
    elif cur is not None and cur[1] and r:
        cur[2].append(r)
name, ix, rows = [b for b in blocks if want in b[0]][occ]
ie, ss = ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"]
runs = []
for k, r in enumerate(rows):
    e = float(r[ie] or 0)
    s = float(r[ss] or 0)
    if runs and runs[-1][1] == e:
        runs[-1][2] += 1
        runs[-1][3] += s
    else:
        runs.append([k, e, 1, s])
tot = sum(e * n for _, e, n, _ in runs)
tots = sum(s for *_, s in runs)
print(name[:100], f"total {tot:.0f} warp instr, {tots:.0f} stall samples")
for k, e, n, s in sorted(runs, key=lambda x: -x[1] * x[2])[:top]:
    src = rows[k][ix["Source"]].strip()[:60]
    print(f"@{k:5d} len {n:4d} x {e:9.0f} = {e*n:11.0f} ({100*e*n/tot:4.1f}%) stalls {100*s/max(tots,1):4.1f}%  {src}")
