timeout 900 python -m pytest tests -m gpu -x -q -k "lsc or signal2sh or sh2signal or functional or kat or cfg1 or cfg3 or ragged or large" 2>&1 | tail -2
for c in cfg1 cfg3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r2k_$c.json 2>/dev/null; echo "$c rc=$?"; done
python - <<'PY'
import json
for c in ["cfg1","cfg3"]:
    d=json.load(open(f"gpurun_out/r2k_{c}.json")); print(c, d["ms_per_step"], d["phase_ms"], d["roofline"]["frac"])
PY
