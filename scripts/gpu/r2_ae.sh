AB_STEPS="--steps 20 --warmup 5" bash scripts/ab_bench.sh "c166885d sm100a" 3
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
