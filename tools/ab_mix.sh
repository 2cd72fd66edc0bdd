#!/bin/bash
# A/B of (library variant, env) pairs under gpurun: tools/ab_mix.sh "name:variant:VAR=v,VAR2=v" ...
# variant "-" = the in-tree library; bench args via BENCH_ARGS
for spec in "$@"; do
  IFS=: read -r name var envs <<< "$spec"
  L=""; [ "$var" != "-" ] && L="HG_LIB_PATH=variants/$var/libhgb200.so"
  env $L ${envs//,/ } timeout 900 python bench.py --no-cpu-baseline $BENCH_ARGS > gpurun_out/abm_$name.json 2> gpurun_out/abm_$name.err
done
python - "$@" <<'PY'
import json, sys
for spec in sys.argv[1:]:
    v = spec.split(":")[0]
    try:
        d = json.loads(open(f"gpurun_out/abm_{v}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(v, "failed", e); continue
    tl = d["timeline_ms"]
    print(f"{v:10s} value {d['value']:.4g} e2e {d['e2e']['value']:.4g} ms {d['ms_per_step']:.4f} "
          f"pruned {tl.get('pruned')} fwd0 {tl.get('forward0')} samp {tl.get('next_sampled (side)')} "
          f"c1 {tl.get('cache_update1 (side)')} sgd {tl.get('sgd')} joined {tl.get('joined')}")
PY
