#!/bin/bash
# Round-2 evidence pass on one B200 (run under gpurun from the repo root):
# launch list of the C2 step, one `ncu --set full` launch per kernel family
# VERDICT r01 asked for, and compute-sanitizer over a GPU test subset.
# Outputs land in gpurun_out/r02prof/ (copied to profiles/r02/ afterwards).
set -u
OUT=gpurun_out/r02prof
mkdir -p $OUT
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 900 --csv --log-file $OUT/launches_c2.csv \
    $B > $OUT/launches_bench.log 2>&1
for k in k_transpose_agg k_aggregate k_gather_dz k_tile_scan k_write_rows k_bs_small k_select k_load_rows; do
  ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 40 -c 1 -o $OUT/ncu_${k} -f \
      $B > $OUT/ncu_${k}.log 2>&1
  ncu -i $OUT/ncu_${k}.ncu-rep --page details --csv > $OUT/ncu_${k}_details.csv 2>/dev/null
  ncu -i $OUT/ncu_${k}.ncu-rep --page raw --csv > $OUT/ncu_${k}_raw.csv 2>/dev/null
  rm -f $OUT/ncu_${k}.ncu-rep
done
S=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $S --tool memcheck --leak-check no --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" \
    > $OUT/sanitizer_memcheck_smoke.log 2>&1; echo "memcheck smoke rc=$?" >> $OUT/sanitizer_summary.txt
timeout 1500 $S --tool racecheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" \
    > $OUT/sanitizer_racecheck_smoke.log 2>&1; echo "racecheck smoke rc=$?" >> $OUT/sanitizer_summary.txt
timeout 1500 $S --tool synccheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" \
    > $OUT/sanitizer_synccheck_smoke.log 2>&1; echo "synccheck smoke rc=$?" >> $OUT/sanitizer_summary.txt
timeout 2400 $S --tool memcheck --leak-check no --error-exitcode 9 python -m pytest -q -x \
    tests/test_gpu_sampler.py tests/test_gpu_cache.py tests/test_gpu_prune_nn.py tests/test_gpu_tcgemm.py \
    "tests/test_gpu_shardcache.py::test_world1_sharded_cache_is_the_local_cache" \
    > $OUT/sanitizer_memcheck_tests.log 2>&1; echo "memcheck tests rc=$?" >> $OUT/sanitizer_summary.txt
cat $OUT/sanitizer_summary.txt
