#!/bin/bash
# Round-end refresh on the GPU box (run under gpurun): GPU tests, smoke, the
# bench lines of every config, the reference arm, and the c2 profiling pass.
set -u
O=gpurun_out/refresh
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_c2.log 2>&1; tail -1 $O/bench_c2.log > $O/bench_c2.json
for c in c3 c5 c4s; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.log 2>&1; tail -1 $O/bench_$c.log > $O/bench_$c.json
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; tail -1 $O/bench_ref.log > $O/bench_ref.json
[ "${SKIP_PROFILE:-0}" = 1 ] || bash tools/profile.sh c2 k_load_rows k_aggregate
