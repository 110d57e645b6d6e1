for r in 1 2 3; do for t in base sm100a; do
  DELIMIT_LIB=paper_1808_01517_b200/libdelimit_$t.so timeout 300 python bench.py --config cfg5 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab5.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab5.json'));print('$t cfg5', round(d['ms_per_step'],3), d.get('roofline',{}).get('launch_ms'), d['clocks']['sm_mhz'])"
done; done
timeout 900 python -m pytest tests -m gpu -x -q -k "mse or MSE or stack or Stack or cfg5 or network" 2>&1 | tail -2
timeout 300 python scripts/ncu_chain.py 3 && echo plain ok
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain2h -s 2 -c 1 -f -o gpurun_out/r2y_chain python scripts/ncu_chain.py 3 > gpurun_out/r2y_ncu.log 2>&1; echo ncu rc=$?
