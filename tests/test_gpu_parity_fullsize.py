"""Parity at the BASELINE configurations' exact sizes (BASELINE.json configs[0..3]).

Every voxel of every output is compared, not a sample:

* cfg4 -- fused Signal2SH -> LSC 3->3 -> SH2Signal fwd + bwd on (1, 270, 145, 174, 145):
  y, dx, dW and db against an independent float64 torch computation over all 3,658,350
  voxels (chunked), whose operators come from the oracle port (oracle/port.py: fit operator
  fitting.py:108-149, ring resample / refit lsc.py:87-135, basis shcore.py:112-166).  The
  fp64 composite is itself checked against port.chain_forward / chain_backward (the
  structured reference algorithm, resample -> ring reduce -> refit) on a voxel sample, and
  every voxel of the last, partial 128-voxel tile (3,658,350 = 28,580 * 128 + 110) is checked
  against the port directly.
* cfg2 -- Signal2SH -> SH2Signal round trip on the same volume, fwd + bwd, fp64 torch.
* cfg3 -- LocalSphericalConvolution 1->1 on (4, 45, 32, 32, 32), fwd + bwd, vs the port.
* cfg1 -- Signal2SH on (1, 90, 32, 32, 32) vs the port.
* cfg5 -- one subject of the training step (2 stacked LSC layers, fused MSE, g-only adjoint): the loss and
  every layer's dW / db over every voxel, float64.

Tolerances (north_star): normwise max|got - ref| / max|ref| <= 1e-5 for SH coefficients and
signals (cfg1, cfg2), <= 1e-4 for LSC outputs and all LSC-chain gradients (cfg3, cfg4).
"""

import math

import numpy as np
import pytest
import torch

import paper_1808_01517_b200 as dl
from paper_1808_01517_b200.directions import unit_sphere_directions
from oracle import port

TOL_SH = 1e-5
TOL_LSC = 1e-4
HCP = (145, 174, 145)
ORDER, LAM, NDIR, SHELLS = 8, 0.006, 90, 3
CHUNK = 1 << 18


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1808_01517_b200._build import build_library

    build_library()
    return torch.device("cuda:0")


def N(t):
    return t.detach().double().cpu().numpy()


class RelErr:
    """Running normwise error max|got - ref| / max|ref| over chunks of one tensor."""

    def __init__(self):
        self.num = 0.0
        self.den = 0.0

    def add(self, got, ref):
        self.num = max(self.num, float((got.double() - ref).abs().max()))
        self.den = max(self.den, float(ref.abs().max()))

    @property
    def value(self):
        return self.num / self.den if self.den > 0 else self.num


def hcp_inputs(dev, seed):
    """Band-limited synthetic signals (phantom.py:77-88) + noise and an N(0,1) upstream gradient."""
    V = int(np.prod(HCP))
    d = unit_sphere_directions(NDIR)
    B = torch.tensor(port.eval_basis(d, ORDER), dtype=torch.float32, device=dev)
    l = torch.tensor(port.degrees(ORDER), dtype=torch.float32, device=dev)
    amp = 0.9 / (1.0 + l * (l + 1.0) / 4.0)
    x = torch.empty((1, SHELLS * NDIR, V), dtype=torch.float32, device=dev)
    for s in range(SHELLS):
        g = torch.Generator(device=dev).manual_seed(seed + s)
        coeffs = (torch.rand((B.shape[1], V), generator=g, device=dev) * 2 - 1) * amp[:, None]
        coeffs[0] = 2.0 * math.sqrt(math.pi)
        x[0, s * NDIR:(s + 1) * NDIR] = B @ coeffs
        x[0, s * NDIR:(s + 1) * NDIR] += 0.02 * torch.randn((NDIR, V), generator=g, device=dev)
        del coeffs
    g = torch.Generator(device=dev).manual_seed(seed + 17)
    dy = torch.randn((1, SHELLS * NDIR, V), generator=g, device=dev)
    return x.view(1, SHELLS * NDIR, *HCP), dy.view(1, SHELLS * NDIR, *HCP)


def chain_operators(d, w, b):
    """float64 operators of the chain from the oracle port: per output shell o and input shell s,
    T[o,s] = B' L_{o,s} M (N x N) and the bias response B' beta bias[o]; plus M, B', P_k, beta."""
    M, _, _ = port.fit_operator(d, ORDER, LAM)
    geo = port.lsc_geometry(d, [5], np.pi / 5, ORDER, ORDER, LAM)
    Bt = port.eval_basis(d, ORDER)
    K = geo["K"]
    R = M.shape[0]
    P = np.stack([geo["refit"] @ geo["resample"][k::K] for k in range(K)])      # (K, R_out, R_in)
    beta = geo["refit"].sum(axis=1)                                             # refit . 1 = 2 sqrt(pi) e0
    so, si = w.shape[0], w.shape[1]
    L = np.einsum("osk,krt->orst", w, P).reshape(so * R, si * R)
    Mb = np.kron(np.eye(si), M)                                                 # block-diagonal M
    Bb = np.kron(np.eye(so), Bt)
    T = Bb @ L @ Mb                                                             # (so*N, si*N)
    y0 = Bb @ np.kron(b, beta)                                                  # bias response
    return dict(M=M, geo=geo, Bt=Bt, P=P, beta=beta, T=T, y0=y0, Mb=Mb, Bb=Bb)


def test_fp64_composite_matches_port():
    """The float64 composite used below equals the structured reference algorithm (CPU, 512 voxels)."""
    d = unit_sphere_directions(NDIR)
    rng = np.random.default_rng(5)
    w = rng.normal(size=(3, 3, 6)) / 18.0
    b = rng.normal(size=3) * 0.1
    ops = chain_operators(d, w, b)
    x = rng.uniform(0.1, 1.3, size=(1, 270, 512, 1, 1))
    dy = rng.normal(size=(1, 270, 512, 1, 1))
    y_port = port.chain_forward(x, ops["M"], ops["geo"], w, b, ops["Bt"], 3)
    dx_port, dW_port, db_port = port.chain_backward(x, dy, ops["M"], ops["geo"], w, ops["Bt"], 3)
    X, DY = x.reshape(270, -1), dy.reshape(270, -1)
    assert port.rel_err(ops["T"] @ X + ops["y0"][:, None], y_port.reshape(270, -1)) <= 1e-12
    assert port.rel_err(ops["T"].T @ DY, dx_port.reshape(270, -1)) <= 1e-12
    G = (ops["Bb"].T @ DY) @ (ops["Mb"] @ X).T
    dW = np.einsum("krt,orst->osk", ops["P"], G.reshape(3, 45, 3, 45))
    db = (ops["Bb"].T @ DY).reshape(3, 45, -1).sum(axis=2) @ ops["beta"]
    assert port.rel_err(dW, dW_port) <= 1e-12
    assert port.rel_err(db, db_port) <= 1e-12


@pytest.mark.gpu
def test_cfg4_hcp_full_volume_fwd_bwd(dev):
    """cfg4 at its exact size: y, dx, dW, db over every voxel against float64."""
    d = unit_sphere_directions(NDIR)
    rng = np.random.default_rng(1)
    w = rng.normal(size=(3, 3, 6)) / 18.0
    b = rng.normal(size=3) * 0.1
    s2sh = dl.Signal2SH(ORDER, d, lb_lambda=LAM).to(dev)
    lsc = dl.LocalSphericalConvolution(3, 3, ORDER, ORDER, d, [5], lb_lambda=LAM, angular_distance=np.pi / 5).to(dev)
    lsc.load_kernel(dl.LscKernel(w, b))
    sh2s = dl.SH2Signal(ORDER, d).to(dev)
    chain = dl.SphericalChain(s2sh, lsc, sh2s)
    assert chain.fused()
    x, dy = hcp_inputs(dev, 1000)
    x.requires_grad_(True)
    for _ in range(2):   # the second call runs with the delayed-scaling state the first one left
        x.grad = None
        lsc.zero_grad(set_to_none=True)
        y = chain(x)
        y.backward(dy)
    torch.cuda.synchronize()
    wq, bq = N(lsc.sconv.weight)[:, :, 0, :], N(lsc.sconv.bias)
    ops = chain_operators(d, wq, bq)
    T = torch.tensor(ops["T"], dtype=torch.float64, device=dev)
    y0 = torch.tensor(ops["y0"], dtype=torch.float64, device=dev)[:, None]
    Mb = torch.tensor(ops["Mb"], dtype=torch.float64, device=dev)
    Bb = torch.tensor(ops["Bb"], dtype=torch.float64, device=dev)
    V = int(np.prod(HCP))
    X, DY = x.detach().view(270, V), dy.view(270, V)
    Y, DX = y.detach().view(270, V), x.grad.view(270, V)
    ey, edx = RelErr(), RelErr()
    G = torch.zeros((135, 135), dtype=torch.float64, device=dev)
    gsum = torch.zeros(135, dtype=torch.float64, device=dev)
    for lo in range(0, V, CHUNK):
        hi = min(V, lo + CHUNK)
        xc, dyc = X[:, lo:hi].double(), DY[:, lo:hi].double()
        ey.add(Y[:, lo:hi], T @ xc + y0)
        edx.add(DX[:, lo:hi], T.T @ dyc)
        g = Bb.T @ dyc
        G += g @ (Mb @ xc).T
        gsum += g.sum(dim=1)
    P = torch.tensor(ops["P"], dtype=torch.float64, device=dev)
    dW_ref = torch.einsum("krt,orst->osk", P, G.view(3, 45, 3, 45))
    db_ref = gsum.view(3, 45) @ torch.tensor(ops["beta"], dtype=torch.float64, device=dev)
    e_dW = port.rel_err(N(lsc.sconv.weight.grad)[:, :, 0, :], N(dW_ref))
    e_db = port.rel_err(N(lsc.sconv.bias.grad), N(db_ref))
    print(f"cfg4 full volume rel err: y {ey.value:.2e} dx {edx.value:.2e} dW {e_dW:.2e} db {e_db:.2e} "
          f"(tolerance {TOL_LSC:g})")
    assert ey.value <= TOL_LSC and edx.value <= TOL_LSC
    assert e_dW <= TOL_LSC and e_db <= TOL_LSC

    # every voxel of the last (partial) tile, directly against the oracle port
    tail = V % 128
    assert tail == 110
    sl = slice(V - tail, V)
    xs = N(X[:, sl]).reshape(1, 270, tail, 1, 1)
    dys = N(DY[:, sl]).reshape(1, 270, tail, 1, 1)
    y_ref = port.chain_forward(xs, ops["M"], ops["geo"], wq, bq, ops["Bt"], 3)
    dx_ref, _, _ = port.chain_backward(xs, dys, ops["M"], ops["geo"], wq, ops["Bt"], 3)
    e_ty = port.rel_err(N(Y[:, sl]).reshape(y_ref.shape), y_ref)
    e_tdx = port.rel_err(N(DX[:, sl]).reshape(dx_ref.shape), dx_ref)
    print(f"cfg4 last tile ({tail} voxels) rel err: y {e_ty:.2e} dx {e_tdx:.2e}")
    assert e_ty <= TOL_LSC and e_tdx <= TOL_LSC


def _round_trip(dev):
    d = unit_sphere_directions(NDIR)
    s2sh = dl.Signal2SH(ORDER, d, lb_lambda=LAM).to(dev)
    sh2s = dl.SH2Signal(ORDER, d).to(dev)
    return d, s2sh, sh2s


@pytest.mark.gpu
def test_cfg2_hcp_round_trip_full_volume(dev):
    """cfg2 at its exact size: the fused Signal2SH -> SH2Signal round trip (dl.RoundTrip), fwd + bwd over every
    voxel against float64."""
    d, s2sh, sh2s = _round_trip(dev)
    x, dy = hcp_inputs(dev, 2000)
    x.requires_grad_(True)
    rt = dl.RoundTrip(s2sh, sh2s)
    assert rt.fused(3)   # one tcgen05 pass per direction, c never reaches HBM
    for _ in range(2):
        x.grad = None
        y = rt(x)
        y.backward(dy)
    torch.cuda.synchronize()
    M, _, _ = port.fit_operator(d, ORDER, LAM)
    Bt = port.eval_basis(d, ORDER)
    Tt = torch.tensor(Bt @ M, dtype=torch.float64, device=dev)     # per shell, N x N
    V = int(np.prod(HCP))
    X, DY = x.detach().view(3, NDIR, V), dy.view(3, NDIR, V)
    Y, DX = y.detach().view(3, NDIR, V), x.grad.view(3, NDIR, V)
    ey, edx = RelErr(), RelErr()
    for s in range(3):
        for lo in range(0, V, CHUNK):
            hi = min(V, lo + CHUNK)
            ey.add(Y[s, :, lo:hi], Tt @ X[s, :, lo:hi].double())
            edx.add(DX[s, :, lo:hi], Tt.T @ DY[s, :, lo:hi].double())
    print(f"cfg2 full volume rel err: y {ey.value:.2e} dx {edx.value:.2e} (tolerance {TOL_SH:g})")
    assert ey.value <= TOL_SH and edx.value <= TOL_SH


@pytest.mark.gpu
def test_cfg3_lsc_batch4_32cubed_vs_port(dev):
    """cfg3 at its exact size: LSC 1->1 ([5] ring, pi/5) fwd + bwd on (4, 45, 32, 32, 32) vs the port."""
    d = unit_sphere_directions(NDIR)
    rng = np.random.default_rng(3)
    w = rng.normal(size=(1, 1, 6)) / 6.0
    b = rng.normal(size=1) * 0.1
    lsc = dl.LocalSphericalConvolution(1, 1, ORDER, ORDER, d, [5], lb_lambda=LAM, angular_distance=np.pi / 5).to(dev)
    lsc.load_kernel(dl.LscKernel(w, b))
    c = np.stack([port.bandlimited_coeffs(np.random.default_rng(10 + i), ORDER, 32 ** 3) for i in range(4)])
    c = np.asarray(c, np.float32).astype(np.float64).reshape(4, 45, 32, 32, 32)
    g = np.asarray(rng.normal(size=(4, 45, 32, 32, 32)), np.float32).astype(np.float64)
    ct = torch.tensor(c, dtype=torch.float32, device=dev, requires_grad=True)
    u = lsc(ct)
    u.backward(torch.tensor(g, dtype=torch.float32, device=dev))
    geo = port.lsc_geometry(d, [5], np.pi / 5, ORDER, ORDER, LAM)
    u_ref = port.lsc_forward(c, w, b, geo)
    dc_ref, dW_ref, db_ref = port.lsc_backward(c, g, w, geo)
    errs = dict(u=port.rel_err(N(u), u_ref), dc=port.rel_err(N(ct.grad), dc_ref),
                dW=port.rel_err(N(lsc.sconv.weight.grad)[:, :, 0, :], dW_ref),
                db=port.rel_err(N(lsc.sconv.bias.grad), db_ref))
    print("cfg3 rel err:", {k: f"{v:.2e}" for k, v in errs.items()}, f"(tolerance {TOL_LSC:g})")
    assert all(v <= TOL_LSC for v in errs.values()), errs


@pytest.mark.gpu
def test_cfg1_signal2sh_32cubed_vs_port(dev):
    """cfg1 at its exact size: Signal2SH(8, 90 dirs) on (1, 90, 32, 32, 32) fwd + bwd vs the port."""
    d = unit_sphere_directions(NDIR)
    s2sh = dl.Signal2SH(ORDER, d, lb_lambda=LAM).to(dev)
    rng = np.random.default_rng(4)
    B = port.eval_basis(d, ORDER)
    x = B @ port.bandlimited_coeffs(rng, ORDER, 32 ** 3) + rng.normal(0, 0.02, size=(90, 32 ** 3))
    x = np.asarray(x, np.float32).astype(np.float64).reshape(1, 90, 32, 32, 32)
    dc = np.asarray(rng.normal(size=(1, 45, 32, 32, 32)), np.float32).astype(np.float64)
    xt = torch.tensor(x, dtype=torch.float32, device=dev, requires_grad=True)
    c = s2sh(xt)
    c.backward(torch.tensor(dc, dtype=torch.float32, device=dev))
    M, _, _ = port.fit_operator(d, ORDER, LAM)
    e_c = port.rel_err(N(c), port.signal_to_sh(x, M, 1))
    e_dx = port.rel_err(N(xt.grad), port.signal_to_sh_adjoint(dc, M, 1))
    print(f"cfg1 rel err: c {e_c:.2e} dx {e_dx:.2e} (tolerance {TOL_SH:g})")
    assert e_c <= TOL_SH and e_dx <= TOL_SH


@pytest.mark.gpu
def test_cfg5_hcp_two_layer_mse_step_full_volume(dev):
    """cfg5's training step on one HCP subject: Signal2SH -> 2 x LSC 3->3 -> SH2Signal, the MSE loss fused into the
    forward kernel and an input that needs no gradient (the g-only adjoint: stage 1 and the Gram planes only).
    The loss and every layer's dW / db over all 3,658,350 voxels against float64."""
    d = unit_sphere_directions(NDIR)
    rng = np.random.default_rng(7)
    ws = [rng.normal(size=(3, 3, 6)) / 18.0 for _ in range(2)]
    bs = [rng.normal(size=3) * 0.1 for _ in range(2)]
    s2sh = dl.Signal2SH(ORDER, d, lb_lambda=LAM).to(dev)
    lscs = []
    for w, b in zip(ws, bs):
        m = dl.LocalSphericalConvolution(3, 3, ORDER, ORDER, d, [5], lb_lambda=LAM, angular_distance=np.pi / 5).to(dev)
        m.load_kernel(dl.LscKernel(w, b))
        lscs.append(m)
    sh2s = dl.SH2Signal(ORDER, d).to(dev)
    net = dl.SphericalChain(s2sh, lscs, sh2s)
    assert net.fused()
    x, _ = hcp_inputs(dev, 2000)
    t, _ = hcp_inputs(dev, 3000)
    for _ in range(2):   # the second call runs with the delayed-scaling state the first one left
        for m in lscs:
            m.zero_grad(set_to_none=True)
        loss = net.mse_loss(x, t)
        loss.backward()
    torch.cuda.synchronize()
    wq = [N(m.sconv.weight)[:, :, 0, :] for m in lscs]
    bq = [N(m.sconv.bias) for m in lscs]
    ops = [chain_operators(d, w, b) for w, b in zip(wq, bq)]
    td = lambda a: torch.tensor(a, dtype=torch.float64, device=dev)   # noqa: E731
    M, Bt, beta, P = ops[0]["M"], ops[0]["Bt"], td(ops[0]["beta"]), td(ops[0]["P"])
    K, R = P.shape[0], M.shape[0]
    L = [td(np.einsum("osk,krt->orst", w, ops[0]["P"]).reshape(3 * R, 3 * R)) for w in wq]
    bias = [td(np.kron(b, ops[0]["beta"]))[:, None] for b in bq]
    Mb, Bb = td(np.kron(np.eye(3), M)), td(np.kron(np.eye(3), Bt))
    V = int(np.prod(HCP))
    X, TT = x.view(270, V), t.view(270, V)
    nel = 270.0 * V
    sq = 0.0
    G2 = torch.zeros((135, 135), dtype=torch.float64, device=dev)
    G1 = torch.zeros((135, 135), dtype=torch.float64, device=dev)
    s2 = torch.zeros(135, dtype=torch.float64, device=dev)
    s1 = torch.zeros(135, dtype=torch.float64, device=dev)
    for lo in range(0, V, CHUNK):
        hi = min(V, lo + CHUNK)
        c = Mb @ X[:, lo:hi].double()
        u1 = L[0] @ c + bias[0]
        u2 = L[1] @ u1 + bias[1]
        r = Bb @ u2 - TT[:, lo:hi].double()
        sq += float((r * r).sum())
        g2 = Bb.T @ (2.0 * r / nel)
        g1 = L[1].T @ g2
        G2 += g2 @ u1.T
        G1 += g1 @ c.T
        s2 += g2.sum(dim=1)
        s1 += g1.sum(dim=1)
    e_loss = abs(float(loss.detach()) - sq / nel) / (sq / nel)
    errs = [e_loss]
    for m, G, gs in ((lscs[0], G1, s1), (lscs[1], G2, s2)):
        dW_ref = torch.einsum("krt,orst->osk", P, G.view(3, R, 3, R))
        db_ref = gs.view(3, R) @ beta
        errs += [port.rel_err(N(m.sconv.weight.grad)[:, :, 0, :], N(dW_ref)), port.rel_err(N(m.sconv.bias.grad), N(db_ref))]
    print("cfg5 one-subject step rel err: loss {:.2e} dW1 {:.2e} db1 {:.2e} dW2 {:.2e} db2 {:.2e}".format(*errs))
    assert e_loss <= TOL_SH
    assert max(errs[1:]) <= TOL_LSC
