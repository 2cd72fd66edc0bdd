"""Print the kernel sequence of an ncu launch-list CSV (optionally a window
starting at the n-th occurrence of a kernel-name substring)."""
import csv
import sys


def load(path):
    hdr, ks = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                ks.append((d["Kernel Name"], float(d["Metric Value"]) / 1000.0))
    return ks


if __name__ == "__main__":
    ks = load(sys.argv[1])
    start = 0
    if len(sys.argv) > 2:
        occ = [i for i, k in enumerate(ks) if sys.argv[2] in k[0]]
        start = occ[int(sys.argv[3]) if len(sys.argv) > 3 else 0]
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    for name, us in ks[start:start + n]:
        print(f"{us:8.1f}  {name[:100]}")
