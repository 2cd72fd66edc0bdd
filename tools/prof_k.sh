#!/bin/bash
# ncu --set full of the launches matching a regex in the C2 step (run under gpurun):
#   tools/prof_k.sh NAME REGEX COUNT [SKIP]  -> gpurun_out/prof/NAME_{details,raw}.csv + launch list
set -u
NAME=$1; RE=$2; C=${3:-6}; S=${4:-60}
OUT=gpurun_out/prof; mkdir -p $OUT
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:"$RE" -s $S -c $C -o $OUT/$NAME -f $B > $OUT/$NAME.log 2>&1
ncu -i $OUT/$NAME.ncu-rep --page details --csv > $OUT/${NAME}_details.csv 2>/dev/null
ncu -i $OUT/$NAME.ncu-rep --page raw --csv > $OUT/${NAME}_raw.csv 2>/dev/null
ncu -i $OUT/$NAME.ncu-rep --page source --csv --print-source sass > $OUT/${NAME}_sass.csv 2>/dev/null
rm -f $OUT/$NAME.ncu-rep
