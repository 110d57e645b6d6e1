set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "mse or stacked" 2>&1 | tail -2
timeout 900 python bench.py --config cfg5 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2e_cfg5.json 2> gpurun_out/r2e_cfg5.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r2e_cfg5.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernel_ms']['fwd_ms'], d['kernel_ms'].get('bwd_ms'))"
python scripts/ncu_chain.py 3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain2h -s 2 -c 2 -f -o gpurun_out/r2e_chain python scripts/ncu_chain.py 3 > gpurun_out/r2e_ncu.log 2>&1; echo ncu rc=$?
