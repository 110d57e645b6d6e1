timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_fullsize.py -x -q -k "without_dx or mse or cfg5 or chain_vs_oracle" 2>&1 | tail -1
for r in 1 2 3; do for t in base sm100a; do
  DELIMIT_LIB=paper_1808_01517_b200/libdelimit_$t.so timeout 300 python bench.py --config cfg5 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab5.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab5.json'));k=d.get('kernel_ms') or {};print('$t cfg5', round(d['ms_per_step'],3), round(k.get('fwd_ms',0),3), round(k.get('bwd_ms',0),3), d['clocks']['sm_mhz'])"
done; done
