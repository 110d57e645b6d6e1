timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in cfg1 cfg3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > gpurun_out/r2j_$c.json 2>/dev/null; echo "$c rc=$?"; done
python - <<'PY'
import json
for c in ["cfg1","cfg3"]:
    d=json.load(open(f"gpurun_out/r2j_{c}.json")); print(c, d["ms_per_step"], d["phase_ms"], d["roofline"]["frac"])
PY
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2j_cfg3_launches.csv python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu --no-e2e --no-clocks > /dev/null 2>&1; echo ncu rc=$?
