timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "stacked or mse or without_dx" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_bench_contract.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2u.json 2> gpurun_out/r2u.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r2u.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['phase_ms'], d['kernel_ms']['fwd_ms'])"
