set -u
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
HG_INPLACE_HITS=1 timeout 900 python -m pytest tests/test_gpu_shardcache.py tests/test_gpu_trainer.py tests/test_gpu_dist.py -m gpu -q -x 2>&1 | tail -2
HG_INPLACE_HITS=0 timeout 900 python -m pytest tests/test_gpu_trainer.py -m gpu -q -x 2>&1 | tail -2
BENCH_ARGS="--steps 300" bash tools/ab_env.sh "auto:" "never:HG_INPLACE_HITS=0" 2>&1 | tail -2
