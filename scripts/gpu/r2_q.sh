DELIMIT_LIB=paper_1808_01517_b200/libdelimit_cv3.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_chain_vs_oracle or mse" 2>&1 | tail -1
DELIMIT_LIB=paper_1808_01517_b200/libdelimit_out3.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_chain_vs_oracle or mse" 2>&1 | tail -1
bash scripts/ab_bench.sh "sm100a cv3 out3" 3
AB_ARGS="--config cfg5" bash scripts/ab_bench.sh "sm100a out3" 1
