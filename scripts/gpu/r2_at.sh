timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2 3; do for t in base sm100a; do
  DELIMIT_LIB=paper_1808_01517_b200/libdelimit_$t.so timeout 300 python bench.py --config cfg5 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab5.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab5.json'));k=d.get('kernel_ms') or {};print('$t cfg5', round(d['ms_per_step'],3), round(k.get('fwd_ms',0),3), round(k.get('bwd_ms',0),3), d['clocks']['sm_mhz'])"
done; done
AB_STEPS="--steps 20 --warmup 5" bash scripts/ab_bench.sh "base sm100a" 2
