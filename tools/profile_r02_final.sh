#!/bin/bash
# Round-2 final evidence pass on one B200 (run under gpurun from the repo root):
# the C2 launch list, `ncu --set full` of each hot kernel family (all layers
# of a step where they differ), and compute-sanitizer over the GPU tests that
# drive the kernels rewritten this round. Outputs: gpurun_out/r02final/.
set -u
OUT=gpurun_out/r02final
mkdir -p $OUT
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv --log-file $OUT/launches_c2.csv \
    $B > $OUT/launches_bench.log 2>&1
cap() {   # name regex count skip
  ncu --set full --clock-control none --import-source on -k regex:"$2" -s $4 -c $3 -o $OUT/ncu_$1 -f $B \
      > $OUT/ncu_$1.log 2>&1
  ncu -i $OUT/ncu_$1.ncu-rep --page details --csv > $OUT/ncu_$1_details.csv 2>/dev/null
  ncu -i $OUT/ncu_$1.ncu-rep --page raw --csv > $OUT/ncu_$1_raw.csv 2>/dev/null
  rm -f $OUT/ncu_$1.ncu-rep
}
cap k_select_all "k_select_all" 3 30
cap k_aggregate "^k_aggregate" 3 30
cap k_transpose_agg "k_transpose_agg" 2 20
cap k_bs "k_bs_|k_norm_keys" 12 60
cap k_write_rows "k_write_rows" 2 20
cap k_tsgemm "k_tsgemm" 8 60
cap k_plan_order "k_plan|k_order|k_pick" 9 30
S=/usr/local/cuda/bin/compute-sanitizer
: > $OUT/sanitizer_summary.txt
timeout 1500 $S --tool memcheck --leak-check no --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" \
    > $OUT/sanitizer_memcheck_smoke.log 2>&1; echo "memcheck smoke rc=$?" >> $OUT/sanitizer_summary.txt
timeout 1500 $S --tool racecheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" \
    > $OUT/sanitizer_racecheck_smoke.log 2>&1; echo "racecheck smoke rc=$?" >> $OUT/sanitizer_summary.txt
timeout 1500 $S --tool synccheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" \
    > $OUT/sanitizer_synccheck_smoke.log 2>&1; echo "synccheck smoke rc=$?" >> $OUT/sanitizer_summary.txt
timeout 2400 $S --tool memcheck --leak-check no --error-exitcode 9 python -m pytest -q -x \
    tests/test_gpu_sampler.py tests/test_gpu_cache.py tests/test_gpu_prune_nn.py \
    "tests/test_gpu_shardcache.py::test_world1_sharded_cache_is_the_local_cache" \
    > $OUT/sanitizer_memcheck_tests.log 2>&1; echo "memcheck tests rc=$?" >> $OUT/sanitizer_summary.txt
timeout 1500 $S --tool racecheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_sampler.py tests/test_gpu_cache.py \
    > $OUT/sanitizer_racecheck_tests.log 2>&1; echo "racecheck sampler+cache tests rc=$?" >> $OUT/sanitizer_summary.txt
cat $OUT/sanitizer_summary.txt
