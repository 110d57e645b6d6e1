AB_STEPS="--steps 20 --warmup 5" bash scripts/ab_bench.sh "sm100a hp" 4
