timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_ingest.py -x -q 2>&1 | tail -2
AB_STEPS="--steps 20 --warmup 5" bash scripts/ab_bench.sh "sm100a a91 r1" 3
