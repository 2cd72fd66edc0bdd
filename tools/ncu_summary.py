"""Summarise an ncu --page details CSV: one line per launch (kernel, duration, key metrics)."""
import csv
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Issued Ipc Active", "Achieved Occupancy",
        "Eligible Warps Per Scheduler", "No Eligible", "Registers Per Thread", "Grid Size", "Block Size",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Avg. Active Threads Per Warp"]
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
cur = None
out = {}
order = []
for r in rows[1:]:
    key = (r[ix["ID"]], r[ix["Kernel Name"]][:60])
    if key not in out:
        out[key] = {}
        order.append(key)
    n = r[ix["Metric Name"]]
    if n in KEYS and n not in out[key]:
        out[key][n] = r[ix["Metric Value"]] + " " + r[ix["Metric Unit"]]
for k in order:
    print(k[0], k[1], "|", "; ".join(f"{n}={v}" for n, v in out[k].items()))
