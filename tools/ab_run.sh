set -u
timeout 900 python -m pytest tests/test_gpu_trainer.py -q -x -k "wide or lockstep" 2>&1 | tail -2
for v in wide2 wide1; do HG_LIB_PATH=variants/$v/libhgb200.so timeout 900 python -m pytest tests/test_gpu_trainer.py -q -x -k "lockstep and not wide" 2>&1 | tail -1; done
bash tools/ab_bench.sh "default wb16 nowide" --config c4s --steps 200 2>&1 | tail -6
bash tools/ab_bench.sh "default wide2 wide1" --steps 300 2>&1 | tail -6
