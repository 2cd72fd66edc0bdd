set -u
BENCH_ARGS="--steps 200 --config c3" bash tools/ab_env.sh "c3auto:" "c3inpl:HG_INPLACE_HITS=1" "c3auto2:" "c3inpl2:HG_INPLACE_HITS=1" 2>&1 | tail -4
BENCH_ARGS="--steps 200 --config c4s" bash tools/ab_env.sh "c4auto:" "c4inpl:HG_INPLACE_HITS=1" 2>&1 | tail -2
