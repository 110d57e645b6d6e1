# round 2, call c: GPU suite, Gram precision, benches, launch list of the default bench command
set -x
timeout 600 python scripts/gram_precision.py 2>&1 | tail -12
timeout 1500 python -m pytest tests -m gpu -x -q -s -k "fullsize or distributed or round_trip or 256x256 or timer" 2>&1 | grep -E "rel err|passed|failed|Error|error" | tail -30
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in cfg4 cfg2 cfg5 cfg1 cfg3; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r2c_$c.json 2> gpurun_out/r2c_$c.err; echo "$c rc=$?"
  tail -c 300 gpurun_out/r2c_$c.err
done
python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 420 --csv --log-file gpurun_out/r2c_launches.csv python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_ncu.log 2>&1; echo "ncu rc=$?"
