#!/bin/bash
# A/B of runtime switches on one box (run under gpurun):
#   tools/ab_env.sh "base:" "sel296:HG_SEL_BLOCKS=296" "prio:HG_NODE_PRIO=1" ...
# each spec is name:VAR=val,VAR2=val (empty = defaults); extra bench args via BENCH_ARGS
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  env ${envs//,/ } timeout 900 python bench.py --no-cpu-baseline $BENCH_ARGS > gpurun_out/abe_$name.json 2> gpurun_out/abe_$name.err
done
python - "$@" <<'PY'
import json, sys
for spec in sys.argv[1:]:
    v = spec.split(":")[0]
    try:
        d = json.loads(open(f"gpurun_out/abe_{v}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(v, "failed", e); continue
    tl = d["timeline_ms"]
    print(f"{v:10s} value {d['value']:.4g} e2e {d['e2e']['value']:.4g} ms {d['ms_per_step']:.4f} "
          f"select {d['per_kernel']['k_select']['ms_per_step']:.4f} samp {tl.get('next_sampled (side)')} "
          f"c1 {tl.get('cache_update1 (side)')} sgd {tl.get('sgd')} joined {tl.get('joined')} "
          f"sus {d['sustained']['value']:.4g} ({d['sustained']['seconds']:.2f} s, caps {d['sustained'].get('graph_captures')})")
PY
