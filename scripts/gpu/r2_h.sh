DELIMIT_LIB=paper_1808_01517_b200/libdelimit_d1e.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chain" 2>&1 | tail -2
bash scripts/ab_bench.sh "sm100a d1e" 3
