timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2v.json 2> gpurun_out/r2v.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r2v.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernel_ms'], d['clocks'])"
