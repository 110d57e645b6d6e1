# round 2, call b: full GPU suite (incl. full-size parity, 2-rank device test), then every bench config
set -x
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -x -q -s -k "fullsize or distributed or round_trip or 256x256" 2>&1 | grep -E "rel err|passed|failed|Error|error" | tail -30
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in cfg4 cfg2 cfg1 cfg3 cfg5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r2b_$c.json 2> gpurun_out/r2b_$c.err; echo "$c rc=$?"
  tail -c 400 gpurun_out/r2b_$c.err
done
python bench.py --gpus 2 --steps 2 --warmup 3; echo "gpus2 rc=$? (expected 2 on a 1-GPU box)"
