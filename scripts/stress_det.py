"""Debug: which fused-chain outputs vary run to run (y, c_mid, dx, dW, db)."""
import sys
import torch
sys.path.insert(0, '/root/repo')
import paper_1808_01517_b200 as dl
from paper_1808_01517_b200.directions import unit_sphere_directions

dev = torch.device('cuda:0')
d = unit_sphere_directions(90)
torch.manual_seed(3)
chain = dl.SphericalChain(dl.Signal2SH(8, d, lb_lambda=0.006).to(dev),
                          dl.LocalSphericalConvolution(3, 3, 8, 8, d, [5]).to(dev), dl.SH2Signal(8, d).to(dev))
V = int(sys.argv[1])
gen = torch.Generator(device=dev).manual_seed(5)
x = torch.rand((1, 270, V, 1, 1), generator=gen, device=dev).requires_grad_(True)
dy = torch.randn((1, 270, V, 1, 1), generator=gen, device=dev)
ref = None
for r in range(int(sys.argv[2])):
    x.grad = None
    chain.zero_grad(set_to_none=True)
    y = chain(x)
    y.backward(dy)
    got = dict(y=y.detach().clone(), dx=x.grad.clone(), dW=chain.lsc.sconv.weight.grad.clone(), db=chain.lsc.sconv.bias.grad.clone())
    if ref is None:
        ref = got
        continue
    for k in got:
        if not torch.equal(got[k], ref[k]):
            diff = (got[k] - ref[k]).abs()
            idx = torch.nonzero(diff.reshape(diff.shape[0], -1) > 0) if diff.dim() > 1 else torch.nonzero(diff > 0)
            print(r, k, 'maxdiff', diff.max().item(), 'count', int((diff > 0).sum()), 'first idx', idx[:3].tolist(), flush=True)
print('done')
