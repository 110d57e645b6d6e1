timeout 900 python -m pytest tests -m gpu -x -q -k "round_trip or cfg2 or fused_chain_vs_oracle" 2>&1 | tail -2
timeout 600 python bench.py --config cfg2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2x.json 2>gpurun_out/r2x.err; echo rc=$?
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2x4.json 2>gpurun_out/r2x4.err; echo rc=$?
python - <<'PY'
import json
for f in ["gpurun_out/r2x.json", "gpurun_out/r2x4.json"]:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d["ms_per_step"], d["phase_ms"], d["kernel_ms"]["fwd_ms"], d["kernel_ms"].get("bwd_ms"), d["roofline"]["frac"], d["clocks"])
PY
