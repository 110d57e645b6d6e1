timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chain" 2>&1 | tail -2
bash scripts/ab_bench.sh "sm100a sm100a:DELIMIT_A2_SPARE=0" 3
