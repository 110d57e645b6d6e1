"""Probe: forward + MSE loss of the cfg5 network, torch's loss on the chain output vs the fused-loss kernel
(argv[1] = 'fused' / 'unfused' / 'both')."""
import math
import sys

import torch

sys.path.insert(0, '/root/repo')
import bench  # noqa: E402
import paper_1808_01517_b200 as dl  # noqa: E402
from paper_1808_01517_b200.directions import unit_sphere_directions  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else 'both'
dev = torch.device('cuda:0')
d = unit_sphere_directions(90)
layers = [dl.LocalSphericalConvolution(3, 3, 8, 8, d, [5], lb_lambda=0.006, angular_distance=math.pi / 5).to(dev)
          for _ in range(2)]
net = dl.SphericalChain(dl.Signal2SH(8, d, lb_lambda=0.006).to(dev), layers, dl.SH2Signal(8, d).to(dev))
x, t = bench.synth_inputs(d, bench.GRID, 0, dev)
for fused in ((True, False) if mode == 'both' else ((mode == 'fused'),)):
    with torch.no_grad():
        for _ in range(3):
            net.mse_loss(x, t, fused=fused)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            loss = net.mse_loss(x, t, fused=fused)
        e1.record()
        torch.cuda.synchronize()
    print('fused' if fused else 'unfused', e0.elapsed_time(e1) / 5, 'ms forward+loss', float(loss),
          'state', [int(v) for v in net.range_state(dev)[0].cpu()])
