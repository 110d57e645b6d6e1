for a in "--steps 10 --warmup 3" "--steps 20 --warmup 5" "--steps 10 --warmup 3" "--steps 40 --warmup 5" "--steps 10 --warmup 3"; do
timeout 600 python bench.py $a --no-cpu --no-e2e > gpurun_out/r2z.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2z.json').read().strip().splitlines()[-1]); k=d['kernel_ms']; print('$a', round(d['ms_per_step'],3), round(k['fwd_ms'],3), [round(x,3) for x in k['fwd_min_max']], d['clocks'].get('sm_min_mhz'), d['clocks'].get('power_w_median'))"
done
nvidia-smi -q -d TEMPERATURE,PERFORMANCE | grep -i "temp\|slowdown\|throttle" | head -20
