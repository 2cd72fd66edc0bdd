set -u
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
bash tools/ab_bench.sh "default prev" --steps 300 2>&1 | grep -v timeline | tail -2
cp gpurun_out/ab_default.json gpurun_out/ab_default_c2.json; cp gpurun_out/ab_prev.json gpurun_out/ab_prev_c2.json
bash tools/ab_bench.sh "default prev" --steps 300 2>&1 | grep -v timeline | tail -2
bash tools/ab_bench.sh "default prev" --config c3 --steps 200 2>&1 | grep -v timeline | tail -2
bash tools/ab_bench.sh "default prev" --config c4s --steps 200 2>&1 | grep -v timeline | tail -2
