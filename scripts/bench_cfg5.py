"""SURVEY cfg5 / BASELINE configs[4]: a small DELIMIT network training step on one HCP-sized subject per GPU.

Signal2SH(8, 90 dirs, lambda .006) -> LSC 3->3 -> LSC 3->3 ([5] ring, pi/5) -> SH2Signal, MSE loss against a
target volume, backward to both LSC layers' weights and biases (no dx), SGD update.  The two LSC layers run
folded through the fused chain kernels (ops.ChainStackFunction).  Prints one JSON line (rank 0); under torchrun
every rank trains on its own subject and the four LSC parameter tensors are all-reduced (distributed.py).
"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1808_01517_b200 as dl  # noqa: E402
from paper_1808_01517_b200.directions import unit_sphere_directions  # noqa: E402


def main(steps=20, warmup=3):
    import torch.distributed as dist

    from paper_1808_01517_b200.distributed import allreduce_gradients, max_over_ranks

    world, rank, local = bench.dist_env()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    d = unit_sphere_directions(90)
    s2sh = dl.Signal2SH(8, d, lb_lambda=0.006).to(dev)
    layers = [dl.LocalSphericalConvolution(3, 3, 8, 8, d, [5], lb_lambda=0.006, angular_distance=math.pi / 5).to(dev)
              for _ in range(2)]
    for k, m in enumerate(layers):
        m.load_kernel(dl.LscKernel(np.random.default_rng(k).normal(size=(3, 3, 6)) / 18,
                                   np.random.default_rng(k).normal(size=3) * 0.1))
    net = dl.SphericalChain(s2sh, layers, dl.SH2Signal(8, d).to(dev))
    x, target = bench.synth_inputs(d, bench.GRID, rank, dev)
    params = [p for m in layers for p in m.parameters()]
    opt = torch.optim.SGD(params, lr=1e-3)
    nvox = x[0, 0].numel()

    fused = os.environ.get("CFG5_UNFUSED_LOSS") is None

    def step():
        opt.zero_grad(set_to_none=True)
        loss = net.mse_loss(x, target, fused=fused)
        loss.backward()
        if world > 1:
            allreduce_gradients(params)
        opt.step()
        return loss

    for _ in range(warmup):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        loss = step()
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, dev)
    if rank == 0:
        print(json.dumps({"metric": "voxels/s, cfg5 training step (Signal2SH -> 2 x LSC -> SH2Signal, MSE, SGD)",
                          "value": world * nvox / (ms / 1e3), "unit": "voxels/s", "n_gpus": world, "steps": steps,
                          "ms_per_step": ms, "loss": float(loss.detach()), "dtype": "f32",
                          "loss_fused": fused,
                          "note": "MSE loss and its gradient inside the forward kernel (CFG5_UNFUSED_LOSS=1: torch's "
                                  "MSE on the chain output); x needs no gradient, so the adjoint is the g-only pass"}))


if __name__ == "__main__":
    main()
