"""Debug: repeat the fused chain backward at a given voxel count; report the first failure."""
import sys
import torch
sys.path.insert(0, '/root/repo')
import paper_1808_01517_b200 as dl
from paper_1808_01517_b200.directions import unit_sphere_directions

dev = torch.device('cuda:0')
d = unit_sphere_directions(90)
chain = dl.SphericalChain(dl.Signal2SH(8, d, lb_lambda=0.006).to(dev),
                          dl.LocalSphericalConvolution(3, 3, 8, 8, d, [5]).to(dev), dl.SH2Signal(8, d).to(dev))
V, reps = int(sys.argv[1]), int(sys.argv[2])
x = torch.rand(1, 270, V, 1, 1, device=dev, requires_grad=True)
dy = torch.randn(1, 270, V, 1, 1, device=dev)
ref = None
for i in range(reps):
    x.grad = None
    for p in chain.parameters():
        p.grad = None
    y = chain(x)
    y.backward(dy)
    torch.cuda.synchronize()
    w = chain.lsc.sconv.weight.grad.clone()
    if ref is None:
        ref = w
    elif not torch.equal(w, ref):
        print('rep', i, 'dW differs', (w - ref).abs().max().item(), flush=True)
print('ok', V, reps, flush=True)
