timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chain or round_trip" 2>&1 | tail -1
AB_STEPS="--steps 20 --warmup 5" bash scripts/ab_bench.sh "sm100a a91" 3
