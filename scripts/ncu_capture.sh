#!/bin/bash
# Launch list + one full ncu capture of each fused kernel (run on the GPU box after bench.py exits 0).
# Usage: scripts/ncu_capture.sh <tag>   -> gpurun_out/<tag>_launches.csv, gpurun_out/<tag>_{chain,gram}.ncu-rep
set -e
tag=${1:-run}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-clocks"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv $B > gpurun_out/${tag}_ncu_launch.log 2>&1
# the fp16 chain pass (chain2h, or chain3v for shapes chain2h does not fit) and its bf16 check pass, and the Gram
ncu --set full --clock-control none --import-source on -k regex:'chain2h|chain3v' -c 3 -f -o gpurun_out/${tag}_chain $B > gpurun_out/${tag}_ncu_chain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gram_tc -c 1 -f -o gpurun_out/${tag}_gram $B > gpurun_out/${tag}_ncu_gram.log 2>&1
echo done
