#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total device time and share (cold-cache, serialised
by ncu, so compare SHARES, not absolute times)."""
import collections
import csv
import re
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    iname, ival = hdr.index("Kernel Name"), hdr.index("Metric Value")
    out = []
    for r in rows[1:]:
        if r[0] == "ID":
            continue
        out.append((r[iname], float(r[ival].replace(",", ""))))
    return out


def short(name):
    name = name.replace("(anonymous namespace)::", "")
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"<([^<>]{0,12})>", r"[\1]", name)
    name = re.sub(r"<.*>", "<..>", name)
    return name.replace("void ", "")[:70]


def main():
    path = sys.argv[1]
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    recs = load(path)[first:]
    tot = collections.defaultdict(lambda: [0, 0.0])
    for n, v in recs:
        k = short(n)
        tot[k][0] += 1
        tot[k][1] += v
    s = sum(v for _, v in tot.values())
    print(f"{'us':>10} {'share':>6} {'n':>5}  kernel")
    for k, (n, v) in sorted(tot.items(), key=lambda x: -x[1][1]):
        print(f"{v / 1e3:10.1f} {100 * v / s:5.1f}% {n:5d}  {k}")
    print(f"total {s / 1e3:.1f} us over {len(recs)} launches")


if __name__ == "__main__":
    main()
