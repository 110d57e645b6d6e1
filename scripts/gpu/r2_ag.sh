AB_STEPS="--steps 20 --warmup 5" bash scripts/ab_bench.sh "base sm100a" 4
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
