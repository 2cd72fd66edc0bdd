set -u
bash tools/ab_bench.sh "default tm6 teb3" --steps 300 2>&1 | grep -v timeline | tail -3
bash tools/ab_bench.sh "default tm6 teb3" --config c3 --steps 200 2>&1 | grep -v timeline | tail -3
