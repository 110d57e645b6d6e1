timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_fullsize.py -x -q 2>&1 | tail -2
AB_STEPS="--steps 20 --warmup 5" bash scripts/ab_bench.sh "base sm100a" 4
