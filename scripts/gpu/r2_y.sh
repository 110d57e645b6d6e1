timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "chain or mse" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2y.json 2>gpurun_out/r2y.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r2y.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['phase_ms'], d['kernel_ms']['fwd_ms'], d['kernel_ms']['bwd_ms'], d['roofline']['frac'])"
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-clocks > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:chain2h -c 4 --csv --log-file gpurun_out/r2y_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-clocks > /dev/null 2>&1; grep -o "chain2h_tc<[0-9]*, [01]>" gpurun_out/r2y_launches.csv | sort | uniq -c
