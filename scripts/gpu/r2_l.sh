python scripts/ncu_chain.py 3 cfg5 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:chain2h -s 2 -c 1 -f -o gpurun_out/r2l_mse python scripts/ncu_chain.py 3 cfg5 > gpurun_out/r2l_ncu_mse.log 2>&1; echo ncu1 rc=$?
python scripts/ncu_chain.py 3 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:chain2h|gram_tc" -s 3 -c 3 -f -o gpurun_out/r2l_chain python scripts/ncu_chain.py 3 > gpurun_out/r2l_ncu_chain.log 2>&1; echo ncu2 rc=$?
