DELIMIT_LIB=paper_1808_01517_b200/libdelimit_u16.so timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "chain" 2>&1 | tail -1
AB_STEPS="--steps 20 --warmup 5" bash scripts/ab_bench.sh "sm100a u16" 4
