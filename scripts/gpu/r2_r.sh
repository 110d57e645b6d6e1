timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "mse or stacked or fused_chain_vs_oracle" 2>&1 | tail -2
AB_ARGS="--config cfg5" bash scripts/ab_bench.sh "sm100a sm100a:DELIMIT_NO_TGTMA=1" 2
