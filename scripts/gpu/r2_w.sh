timeout 900 python -m pytest tests/test_gpu_ingest.py tests/test_gpu_cli.py -x -q 2>&1 | tail -3
timeout 600 python scripts/bench_raw_chain.py 2>&1 | tail -1
DELIMIT_NO_RAWTMA=1 timeout 600 python scripts/bench_raw_chain.py 2>&1 | tail -1
