timeout 300 python scripts/ncu_chain.py 3 && echo plain ok
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain2h -s 2 -c 1 -f -o gpurun_out/r2x_chain python scripts/ncu_chain.py 3 > gpurun_out/r2x_ncu.log 2>&1; echo ncu rc=$?
