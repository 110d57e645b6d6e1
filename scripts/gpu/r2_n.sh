timeout 600 python scripts/bench_raw_chain.py --save 2>&1 | tail -3
timeout 600 python scripts/bench_raw_chain.py > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r2n_raw_launches.csv python scripts/bench_raw_chain.py > /dev/null 2>&1; echo ncu rc=$?
