#!/bin/bash
# A/B timing of library variants / env knobs on one box; alternates the specs R times.
# spec = <lib tag>[:VAR=val[,VAR=val...]]   (libs from scripts/build_variant.sh)
# usage: scripts/ab_bench.sh "A D:DELIMIT_IN_SLOTS=4" [R]   -> summary on stdout
R=${2:-2}
mkdir -p gpurun_out
for r in $(seq 1 $R); do
  for spec in $1; do
    t=${spec%%:*}; envs=""
    [[ "$spec" == *:* ]] && envs=$(echo "${spec#*:}" | tr ',' ' ')
    env $envs DELIMIT_LIB=paper_1808_01517_b200/libdelimit_$t.so timeout 300 python bench.py ${AB_STEPS:---steps 10 --warmup 3} \
      --no-e2e --no-cpu $AB_ARGS > gpurun_out/ab_$r.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_$r.json'));k=d.get('kernel_ms') or {};print('$spec', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()}, 'kern', [round(k.get(x,0),3) for x in ('fwd_ms','bwd_ms','gram_ms')], d['clocks']['sm_mhz'], d['clocks'].get('sm_min_mhz'))" 2>&1 | tail -1
  done
done
