"""Small driver for ncu captures of the fused kernels: cfg4 chain fwd + bwd (HCP size), `reps` times.

    ncu --set full --import-source on -k regex:chain2h -s 2 -c 2 -o ... python scripts/ncu_chain.py
(with -s 2: skips the first fwd + adjoint launches, which settle the fp16 scale)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main(reps=3, cfg="cfg4"):
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    if cfg == "cfg5":
        import paper_1808_01517_b200 as dl
        dirs, s2sh, layers, sh2s = bench.chain_modules(dev, layers=2)
        net = dl.SphericalChain(s2sh, layers, sh2s)
        x = bench.synth_signal(dirs, bench.GRID, 0, dev)
        t = bench.synth_signal(dirs, bench.GRID, 1, dev)
        for _ in range(reps):
            net.mse_loss(x, t).backward()
    else:
        _, _, chain = bench.build_model(dev)
        x, dy = bench.synth_inputs(chain.s2sh.operators[0].gradients, bench.GRID, 0, dev)
        x.requires_grad_(True)
        for _ in range(reps):
            chain(x).backward(dy)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 3, sys.argv[2] if len(sys.argv) > 2 else "cfg4")
