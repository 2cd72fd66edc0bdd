#!/bin/bash
# Round-2 bench lines on one B200 (run under gpurun): C2 (the driver's default
# line), C3 / C5 / C4s, the reference arm, and two ranks sharing the GPU with
# the owner-sharded cache (C1). Outputs: gpurun_out/r02bench/.
set -u
OUT=gpurun_out/r02bench; mkdir -p $OUT
timeout 1200 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
for c in c3 c5 c4s; do timeout 1500 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; done
timeout 1200 python bench.py --impl reference > $OUT/bench_reference_arm.json 2> $OUT/bench_reference_arm.err
HG_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus 2 --config c1 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_2ranks_1gpu_c1_owner_cache.json \
    2> $OUT/bench_2ranks.err
for f in $OUT/*.json; do echo "$f: $(tail -1 $f | cut -c1-200)"; done
