set -u
bash tools/ab_bench.sh "default s3a s3b s3d default" --steps 300 2>&1 | grep -v timeline | tail -5
