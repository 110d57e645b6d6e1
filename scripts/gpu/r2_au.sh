DELIMIT_LIB=paper_1808_01517_b200/libdelimit_cv3.so timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
AB_STEPS="--steps 20 --warmup 5" bash scripts/ab_bench.sh "sm100a cv3" 4
