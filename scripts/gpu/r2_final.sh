# round 2 measurement batch: GPU suite, smoke, every bench config, the reference arm, launch list + ncu captures
# of the chain kernels (each ncu command after the same command exited 0 without ncu).  The .ncu-rep files are
# exported to CSV on the box and deleted (gpurun copies back <= 64 MiB).
set -x
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 > gpurun_out/fin_plain.json 2> gpurun_out/fin_plain.err; echo "plain rc=$?"
for c in cfg2 cfg5 cfg3 cfg1; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/fin_$c.json 2> gpurun_out/fin_$c.err; echo "$c rc=$?"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.json 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 420 --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 20 --warmup 5 > gpurun_out/fin_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python scripts/ncu_chain.py 3 && echo chain ok
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain2h -s 2 -c 1 -f -o /tmp/fin_fwd python scripts/ncu_chain.py 3 > gpurun_out/fin_ncu_fwd.log 2>&1; echo "ncu fwd rc=$?"
ncu -i /tmp/fin_fwd.ncu-rep --page details --csv > gpurun_out/fin_fwd_details.csv 2>/dev/null
ncu -i /tmp/fin_fwd.ncu-rep --page source --csv --print-source sass > gpurun_out/fin_fwd_sass.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k "regex:chain2h|gram_tc" -s 3 -c 3 -f -o /tmp/fin_chain python scripts/ncu_chain.py 3 > gpurun_out/fin_ncu_chain.log 2>&1; echo "ncu chain rc=$?"
ncu -i /tmp/fin_chain.ncu-rep --page details --csv > gpurun_out/fin_chain_details.csv 2>/dev/null
ncu -i /tmp/fin_chain.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active > gpurun_out/fin_chain_raw.csv 2>/dev/null
timeout 300 python scripts/ncu_chain.py 3 cfg5 && echo mse ok
timeout 900 ncu --set full --clock-control none -k regex:chain2h -s 2 -c 1 -f -o /tmp/fin_mse python scripts/ncu_chain.py 3 cfg5 > gpurun_out/fin_ncu_mse.log 2>&1; echo "ncu mse rc=$?"
ncu -i /tmp/fin_mse.ncu-rep --page details --csv > gpurun_out/fin_mse_details.csv 2>/dev/null
ncu -i /tmp/fin_mse.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/fin_mse_raw.csv 2>/dev/null
du -sh gpurun_out
