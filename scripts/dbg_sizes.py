"""Debug: run the fused chain fwd/bwd at several voxel counts (each in a fresh process), report failures."""
import subprocess
import sys

CODE = r'''
import sys, torch
sys.path.insert(0, '/root/repo')
import paper_1808_01517_b200 as dl
from paper_1808_01517_b200.directions import unit_sphere_directions
dev = torch.device('cuda:0')
d = unit_sphere_directions(90)
chain = dl.SphericalChain(dl.Signal2SH(8, d, lb_lambda=0.006).to(dev),
                          dl.LocalSphericalConvolution(3, 3, 8, 8, d, [5]).to(dev), dl.SH2Signal(8, d).to(dev))
V = int(sys.argv[1])
x = torch.rand(1, 270, V, 1, 1, device=dev, requires_grad=True)
y = chain(x); torch.cuda.synchronize(); print('fwd ok', end=' ')
y.backward(torch.randn_like(y)); torch.cuda.synchronize(); print('bwd ok')
'''
for V in sys.argv[1:]:
    r = subprocess.run([sys.executable, '-c', CODE, V], capture_output=True, text=True, timeout=300)
    err = [l for l in r.stderr.splitlines() if 'Error' in l][-1:] if r.returncode else []
    print(V, int(V) % 4, r.stdout.strip(), err, flush=True)
