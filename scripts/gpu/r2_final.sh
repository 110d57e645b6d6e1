# round 2 measurement batch: GPU suite, smoke, every bench config, launch list + full capture of the default command
set -x
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for c in cfg4 cfg2 cfg5 cfg3 cfg1; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/fin_$c.json 2> gpurun_out/fin_$c.err; echo "$c rc=$?"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.json 2>&1; echo "ref rc=$?"
python bench.py --steps 20 --warmup 5 > gpurun_out/fin_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 420 --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 20 --warmup 5 > gpurun_out/fin_ncu.log 2>&1; echo "ncu rc=$?"
