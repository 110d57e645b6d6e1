AB_STEPS="--steps 20 --warmup 5" bash scripts/ab_bench.sh "sm100a ob2 sm100a:DELIMIT_IN_SINGLE=1" 3
