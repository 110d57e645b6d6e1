timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chain or ragged" 2>&1 | tail -2
bash scripts/ab_bench.sh "sm100a prev" 3
