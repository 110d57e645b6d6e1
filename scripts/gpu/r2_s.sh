# multi-rank bench flow on a 1-GPU box: two ranks share cuda:0 with gloo (test mode; NCCL needs distinct GPUs)
for args in "--config cfg4" "--config cfg4 --shard voxels" "--config cfg5 --steps 2"; do
  timeout 300 python bench.py --gpus 2 --dist-backend gloo --steps 5 --warmup 3 --no-cpu $args > gpurun_out/r2s.json 2> gpurun_out/r2s.err
  echo "[$args] rc=$?"; tail -c 600 gpurun_out/r2s.json; grep -i "error" gpurun_out/r2s.err | head -3
done
AB_ARGS="--config cfg5" bash scripts/ab_bench.sh "sm100a pf0" 2
