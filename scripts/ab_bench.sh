#!/bin/bash
# A/B timing of library variants on one box (scripts/build_variant.sh): alternates the variants R times.
# usage: scripts/ab_bench.sh "A B C" [R]   -> gpurun_out/ab_<tag>_<r>.json, summary on stdout
R=${2:-2}
mkdir -p gpurun_out
for r in $(seq 1 $R); do
  for t in $1; do
    DELIMIT_LIB=paper_1808_01517_b200/libdelimit_$t.so timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e \
      --no-cpu > gpurun_out/ab_${t}_$r.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_${t}_$r.json'));print('$t', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()}, d['clocks']['sm_mhz'])"
  done
done
