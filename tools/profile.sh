#!/bin/bash
# Profiling pass on the GPU box (run under gpurun): the ncu launch list of a
# short bench run + one `ncu --set full` capture per named kernel.
#   tools/profile.sh <tag> [kernel regex ...]
set -u
TAG=${1:-c2}; shift || true
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
BENCH="python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-}"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_COUNT:-3000} --csv \
  --log-file $OUT/launches.csv $BENCH > $OUT/launches_bench.log 2>&1
for K in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s ${NCU_SKIP:-12} -c 1 \
    -o $OUT/full_$K $BENCH > $OUT/full_$K.log 2>&1
  ncu -i $OUT/full_$K.ncu-rep --page raw --csv > $OUT/full_${K}_raw.csv 2>/dev/null
  ncu -i $OUT/full_$K.ncu-rep --page details --csv > $OUT/full_${K}_details.csv 2>/dev/null
done
