"""dW / db error of the fused cfg4 backward at the full HCP size vs float64, per Gram wave count.

DELIMIT_GRAM_WAVES = w launches w x 148 Gram CTAs (shorter fp32 TMEM accumulation per partial)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_1808_01517_b200 as dl  # noqa: E402
from paper_1808_01517_b200.directions import unit_sphere_directions  # noqa: E402
from oracle import port  # noqa: E402
from test_gpu_parity_fullsize import chain_operators, hcp_inputs, N, HCP, CHUNK  # noqa: E402

dev = torch.device("cuda:0")
d = unit_sphere_directions(90)
rng = np.random.default_rng(1)
w = rng.normal(size=(3, 3, 6)) / 18.0
b = rng.normal(size=3) * 0.1
s2sh = dl.Signal2SH(8, d, lb_lambda=0.006).to(dev)
lsc = dl.LocalSphericalConvolution(3, 3, 8, 8, d, [5], lb_lambda=0.006, angular_distance=np.pi / 5).to(dev)
lsc.load_kernel(dl.LscKernel(w, b))
chain = dl.SphericalChain(s2sh, lsc, dl.SH2Signal(8, d).to(dev))
x, dy = hcp_inputs(dev, 1000)
V = int(np.prod(HCP))
wq, bq = N(lsc.sconv.weight)[:, :, 0, :], N(lsc.sconv.bias)
ops = chain_operators(d, wq, bq)
Mb = torch.tensor(ops["Mb"], dtype=torch.float64, device=dev)
Bb = torch.tensor(ops["Bb"], dtype=torch.float64, device=dev)
X, DY = x.view(270, V), dy.view(270, V)
G = torch.zeros((135, 135), dtype=torch.float64, device=dev)
gsum = torch.zeros(135, dtype=torch.float64, device=dev)
for lo in range(0, V, CHUNK):
    hi = min(V, lo + CHUNK)
    g = Bb.T @ DY[:, lo:hi].double()
    G += g @ (Mb @ X[:, lo:hi].double()).T
    gsum += g.sum(dim=1)
P = torch.tensor(ops["P"], dtype=torch.float64, device=dev)
dW_ref = N(torch.einsum("krt,orst->osk", P, G.view(3, 45, 3, 45)))
db_ref = N(gsum.view(3, 45) @ torch.tensor(ops["beta"], dtype=torch.float64, device=dev))
print("max|dW_ref|", np.abs(dW_ref).max(), "max|db_ref|", np.abs(db_ref).max())
for waves in (1, 2, 4, 8):
    os.environ["DELIMIT_GRAM_WAVES"] = str(waves)
    for rep in range(2):
        lsc.zero_grad(set_to_none=True)
        y = chain(x)
        y.backward(dy)
        torch.cuda.synchronize()
        e_w = port.rel_err(N(lsc.sconv.weight.grad)[:, :, 0, :], dW_ref)
        e_b = port.rel_err(N(lsc.sconv.bias.grad), db_ref)
        print(f"waves {waves} rep {rep}: dW {e_w:.3e} db {e_b:.3e}")
    # timing of the backward at this wave count
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    y = chain(x)
    torch.cuda.synchronize()
    s0.record()
    y.backward(dy)
    s1.record()
    torch.cuda.synchronize()
    print(f"waves {waves}: backward {s0.elapsed_time(s1):.3f} ms")

# the two-term bf16 representation alone (float64 accumulation): how much of the error is the operand split
Ge = torch.zeros((135, 135), dtype=torch.float64, device=dev)
for lo in range(0, V, CHUNK):
    hi = min(V, lo + CHUNK)
    g = (Bb.T @ DY[:, lo:hi].double()).float()
    c = (Mb @ X[:, lo:hi].double()).float()
    gh = g.bfloat16().float(); gl = (g - gh).bfloat16().float()
    ch = c.bfloat16().float(); cl = (c - ch).bfloat16().float()
    gh, gl, ch, cl = gh.double(), gl.double(), ch.double(), cl.double()
    Ge += gh @ ch.T + gh @ cl.T + gl @ ch.T
dW_e = N(torch.einsum("krt,orst->osk", P, Ge.view(3, 45, 3, 45)))
print(f"bf16x2 operands, float64 accumulation: dW {port.rel_err(dW_e, dW_ref):.3e}")
