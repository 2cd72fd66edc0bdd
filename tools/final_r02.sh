#!/bin/bash
# Round-2 closing evidence on one B200 (run under gpurun from the repo root):
# GPU suite + smoke, the C2 launch list, ncu --set full of the kernels changed
# since the last capture (tcgen05 GEMM epilogue, layer-0 / in-place-hit
# aggregation at C2, layer-0 aggregation at C3 and C4s), traffic.json from
# those captures, then every bench line, the reference arm and the 2-rank
# owner-sharded-cache line, and compute-sanitizer over the changed paths.
# Outputs: gpurun_out/final/.
set -u
OUT=gpurun_out/final
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -1 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
    --log-file $OUT/launches_c2.csv $B > $OUT/launches_bench.log 2>&1
cap() {   # name regex count skip [bench args]
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $4 -c $3 -o $OUT/ncu_$1 -f \
      $B ${5:-} > $OUT/ncu_$1.log 2>&1
  ncu -i $OUT/ncu_$1.ncu-rep --page details --csv > $OUT/ncu_$1_details.csv 2>/dev/null
  ncu -i $OUT/ncu_$1.ncu-rep --page raw --csv > $OUT/ncu_$1_raw.csv 2>/dev/null
  rm -f $OUT/ncu_$1.ncu-rep
}
if [ "${SKIP_NCU:-0}" != 1 ]; then
cap k_aggregate_c2 "^k_aggregate" 3 30
cap k_tsgemm_c2 "k_tsgemm" 8 60
cap k_aggregate_c3 "^k_aggregate" 1 30 "--config c3"
cap k_aggregate_c4s "^k_aggregate" 1 30 "--config c4s"
python - <<'PY'
import csv, json
out = {}
for cfg in ("c2", "c3", "c4s"):
    p = f"gpurun_out/final/ncu_k_aggregate_{cfg}_raw.csv"
    try:
        rows = [r for r in csv.reader(open(p))]
    except OSError:
        continue
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    def val(d, u, k):
        return float(d[k].replace(",", "")) * scale.get(u[k], 1.0)
    for r in rows[2:]:
        if len(r) == len(hdr) and "k_aggregate" in r[hdr.index("Kernel Name")]:
            d, u = dict(zip(hdr, r)), dict(zip(hdr, units))
            rd = val(d, u, "dram__bytes_read.sum")
            wr = val(d, u, "dram__bytes_write.sum")
            out[cfg] = {"kernel": "k_aggregate_rows", "kernel_name": d["Kernel Name"][:80],
                        "dram_bytes_read": rd, "dram_bytes_write": wr,
                        "duration_us": float(d["gpu__time_duration.sum"]), "traffic_bytes": rd + wr,
                        "capture": f"ncu --set full --clock-control none -k regex:^k_aggregate -s 30 python bench.py "
                                   f"--steps 4 --warmup 3 --no-cpu-baseline --config {cfg} (first captured launch = "
                                   f"the layer-0 kernel; profiles/r02/final/ncu_k_aggregate_{cfg}_raw.csv, "
                                   f"tools/final_r02.sh)"}
            break
json.dump(out, open("profiles/r02/traffic.json", "w"), indent=1)
json.dump(out, open("gpurun_out/final/traffic.json", "w"), indent=1)
print("traffic", {k: (v["kernel_name"][:40], v["traffic_bytes"]) for k, v in out.items()})
PY
fi
timeout 1200 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
for c in c3 c5 c4s; do timeout 1500 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; done
timeout 1200 python bench.py --impl reference > $OUT/bench_reference_arm.json 2> $OUT/bench_reference_arm.err
HG_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus 2 --config c1 --steps 20 --warmup 3 --no-cpu-baseline \
    > $OUT/bench_2ranks_1gpu_c1_owner_cache.json 2> $OUT/bench_2ranks.err
for f in $OUT/bench_*.json; do echo "$f: $(tail -1 $f | cut -c1-160)"; done
# compute-sanitizer: closed on the GPU pool at the end of round 2 (the last
# clean runs are in profiles/r02/sanitizer/, tools/profile_r02_final.sh)
