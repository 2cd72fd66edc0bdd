#!/bin/bash
# sampler A/B under gpurun: GPU sampler/trainer tests, then bench per HG_SEL_LANE_MAX value
python -m pytest tests -x -q -m gpu -k "sampler or trainer or c1 or c2 or lockstep or gat" > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
for v in ${LANES:-0 128 0 128}; do
  HG_SEL_LANE_MAX=$v timeout 600 python bench.py --no-cpu-baseline --steps 200 --warmup 20 > gpurun_out/lane_$v.json 2>gpurun_out/lane_$v.err
  python - $v <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/lane_{sys.argv[1]}.json").read().strip().splitlines()[-1])
pk = {k: (round(x["ms_per_step"], 4), x["launches"]) for k, x in d["per_kernel"].items() if x["launches"]}
print(sys.argv[1], round(d["value"]), round(d["e2e"]["value"]), round(d["ms_per_step"], 4),
      d["timeline_ms"]["next_sampled (side)"], pk.get("k_select"))
PY
done
