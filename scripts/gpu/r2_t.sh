timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2t_g.json 2> gpurun_out/r2t_g.err; echo rc=$?
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e --no-graph > gpurun_out/r2t_e.json 2> gpurun_out/r2t_e.err; echo rc=$?
python - <<'PY'
import json
for f in ["gpurun_out/r2t_g.json","gpurun_out/r2t_e.json"]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d["ms_per_step"], d["phase_ms"], d["kernel_ms"]["fwd_ms"], d["reconcile"]["ok"], d["gpu_launches"])
    except Exception as e: print(f, "ERR", e)
PY
tail -5 gpurun_out/r2t_g.err
