set -u
timeout 900 python -m pytest tests/test_gpu_tcgemm.py tests/test_gpu_trainer.py tests/test_gpu_gat.py -q -x 2>&1 | tail -1
bash tools/ab_bench.sh "default st4 st6 default st4" --steps 300 2>&1 | grep -v timeline | tail -5
