# multi-rank bench flow on a 1-GPU box: two ranks share cuda:0 with gloo (test mode; NCCL needs distinct GPUs)
for args in "--config cfg4" "--config cfg4 --shard voxels" "--config cfg2" "--config cfg5 --steps 2"; do
  timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 5 --warmup 3 --no-cpu $args > gpurun_out/r2s.json 2> gpurun_out/r2s.err
  echo "[$args] rc=$?"; tail -c 700 gpurun_out/r2s.json; grep -i "error\|traceback" gpurun_out/r2s.err | head -5
done
