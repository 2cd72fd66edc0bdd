set -u
bash tools/ab_bench.sh "default bh8" --config c3 --steps 200 2>&1 | tail -4
