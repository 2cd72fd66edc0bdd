set -u
timeout 900 python -m pytest tests/test_gpu_tcgemm.py tests/test_gpu_trainer.py tests/test_gpu_prune_nn.py -q -x 2>&1 | tail -2
bash tools/ab_bench.sh "default li0 li_eb8 li_eb2" --steps 300 2>&1 | tail -8
