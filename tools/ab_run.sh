set -u
timeout 900 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_trainer.py -q -x 2>&1 | tail -1
BENCH_ARGS="--steps 200 --config c4s" bash tools/ab_env.sh "c4auto:" "c4s444:HG_SEL_BLOCKS=444" "c4auto2:" "c4s444b:HG_SEL_BLOCKS=444" 2>&1 | tail -4
BENCH_ARGS="--steps 200 --config c3" bash tools/ab_env.sh "c3auto:" 2>&1 | tail -1
BENCH_ARGS="--steps 300" bash tools/ab_env.sh "c2auto:" 2>&1 | tail -1
