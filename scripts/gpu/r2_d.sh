set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "mse or stacked or scale_history" 2>&1 | tail -3
timeout 900 python bench.py --config cfg5 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2d_cfg5.json 2> gpurun_out/r2d_cfg5.err; echo rc=$?
DELIMIT_NO_TRING=1 timeout 900 python bench.py --config cfg5 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2d_cfg5_notring.json 2>&1; echo rc=$?
python - <<'PY'
import json
for f in ["gpurun_out/r2d_cfg5.json", "gpurun_out/r2d_cfg5_notring.json"]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["ms_per_step"], d["kernel_ms"]["fwd_ms"], d["kernel_ms"].get("bwd_ms"))
PY
