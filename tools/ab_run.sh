set -u
timeout 900 python -m pytest tests/test_gpu_gat.py -q -x 2>&1 | tail -1
bash tools/ab_bench.sh "default prev" --config c5 --steps 100 2>&1 | grep -v timeline | tail -2
