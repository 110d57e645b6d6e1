timeout 900 python -m pytest tests/test_gpu_ingest.py tests/test_gpu_cli.py -x -q 2>&1 | tail -3
timeout 600 python scripts/bench_raw_chain.py --save 2>&1 | tail -2
timeout 600 python scripts/bench_raw_chain.py > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:chain|b0_|voxel_scale|ingest|pack|fold|build_op" -c 60 --csv --log-file gpurun_out/r2o_raw_launches.csv python scripts/bench_raw_chain.py > /dev/null 2>&1; echo ncu rc=$?
