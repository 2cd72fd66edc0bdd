#!/bin/bash
# A/B of library variants on one box (run under gpurun): tools/ab_bench.sh "default nopipe minb5" [bench args]
VARS=$1; shift
for v in $VARS; do
  if [ "$v" = default ]; then L=""; else L="HG_LIB_PATH=variants/$v/libhgb200.so"; fi
  env $L timeout 900 python bench.py --no-cpu-baseline "$@" > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
done
python - "$VARS" <<'PY'
import json, sys
for v in sys.argv[1].split():
    try:
        d = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(v, "failed", e); continue
    pk = {k: round(x["ms_per_step"], 4) for k, x in d["per_kernel"].items() if x["launches"]}
    print(f"{v:10s} value {d['value']:.4g} e2e {d['e2e']['value']:.4g} ms {d['ms_per_step']:.4f} "
          f"roof {d['roofline']['frac']:.3f} agg {(d.get('aggregate_roofline') or {}).get('frac', 0):.3f} {pk}")
    print("   timeline", {k: round(x, 3) for k, x in d.get("timeline_ms", {}).items()})
PY
