"""Generate golden vectors by running the REAL reference (sphdwi 0.1.0).

Run in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/golden.npz (float64 arrays).  Inputs are float32-exact
values (generated in float32, upcast), so the CUDA path and the reference see
identical numbers.  Backward vectors are reference-anchored: the reference has
no backward but every layer is exactly linear, so

* J (the Jacobian) is the reference forward applied to identity "voxels";
  dx = J^T dy;
* dW[o,s,k] = <dy, forward(x; weights = e_osk, bias = 0)>   (linear in w);
* db[o]     = <dy, forward(0; weights = 0, bias = e_o)>      (linear in bias).

Nothing here is imported by the product, the tests only read the .npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, os.environ.get("SPHDWI_REF", "/root/reference/pkg/src"))

import sphdwi  # noqa: E402
from sphdwi import (  # noqa: E402
    DwiVolume,
    LscKernel,
    ShBasisSpec,
    ShVolume,
    build_lsc_geometry,
    eval_basis,
    lsc_forward,
    make_fit_operator,
    sh_to_signal,
    signal_to_sh,
    unit_sphere_directions,
)
from sphdwi.phantom import _bandlimited_coeffs  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
TABLES = os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))),
                      "paper_1808_01517_b200", "data", "gradient_tables.npz")


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def rand_dirs(rng, n):
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def lsc_ref(c5, w, b, geom, order_in, shells_in):
    return lsc_forward(ShVolume(data=c5, basis_spec=ShBasisSpec(order_in), shells=shells_in),
                       LscKernel(weights=w, bias=b), geom).data


def chain_ref(x5, op, geom, w, b, target, order, shells_in):
    c = signal_to_sh(DwiVolume(data=x5, shells=shells_in), op)
    u = lsc_forward(c, LscKernel(weights=w, bias=b), geom)
    return sh_to_signal(u, target).data


def jac(fn, nin):
    """Columns of the linear map fn (without bias) on identity voxels: (nout, nin)."""
    eye = np.eye(nin).reshape(1, nin, nin, 1, 1)
    return fn(eye)[0].reshape(-1, nin)


def main():
    rng = np.random.default_rng(20240814)
    g = {}
    for n in (30, 60, 90):
        g[f"dirs{n}"] = unit_sphere_directions(n)
    d90 = g["dirs90"]
    d30 = g["dirs30"]

    # ---- basis and operators ----------------------------------------------------
    rd = rand_dirs(rng, 64)
    rd[0] = [0.0, 0.0, 1.0]      # pole
    rd[1] = [0.0, 0.0, -1.0]     # south pole
    g["basis_dirs"] = rd
    for L in (0, 2, 4, 6, 8, 10):
        g[f"basis_o{L}"] = eval_basis(rd, L)
    g["lb_o8"] = sphdwi.laplace_beltrami_diag(8)
    r40 = rand_dirs(rng, 40)
    g["fit_r40"] = r40
    for tag, dirs, L, lam in [("d90_o8_l006", d90, 8, 0.006), ("d30_o4_l0", d30, 4, 0.0),
                              ("d60_o8_l006", g["dirs60"], 8, 0.006), ("r40_o6_l06", r40, 6, 0.06),
                              ("d90_o4_l0", d90, 4, 0.0)]:
        op = make_fit_operator(dirs, L, lam)
        g[f"fit_{tag}"] = op.fit_matrix
        g[f"cond_{tag}"] = np.array(op.cond)
    # rings / tangent frames
    tu = rand_dirs(rng, 16)
    tu[0] = [0.0, 0.0, 1.0]
    tu[1] = [0.3, 0.1, 0.95]
    g["frame_u"] = tu
    g["frame_e1"] = np.stack([sphdwi.tangent_basis(u)[0] for u in tu])
    g["frame_e2"] = np.stack([sphdwi.tangent_basis(u)[1] for u in tu])
    g["ring_u_a05_n6"] = np.stack([sphdwi.ring_directions(u, 0.5, 6) for u in tu])

    geoms = {
        "g90": (d90, [5], np.pi / 5, 8, 8, 0.006),
        "g30r2": (d30, [4, 8], 0.35, 4, 4, 0.0),
        "g30o42": (d30, [5], 0.52, 4, 2, 0.0),
    }
    G = {}
    for tag, args in geoms.items():
        geo = build_lsc_geometry(*args)
        G[tag] = geo
        g[f"{tag}_resample"] = geo.resample_matrix
        g[f"{tag}_refit"] = geo.refit.fit_matrix

    # ---- Signal2SH / SH2Signal, 3 shells x 90 at order 8 -------------------------
    op90 = make_fit_operator(d90, 8, 0.006)
    B90 = eval_basis(d90, 8)
    nv = (4, 4, 4)
    V = int(np.prod(nv))
    xs = []
    for s in range(3):
        cf = _bandlimited_coeffs(np.random.default_rng(1000 + s), 8, 2 * V)
        xs.append((B90 @ cf).reshape(90, 2, V).transpose(1, 0, 2))
    x = np.concatenate(xs, axis=1) + np.random.default_rng(7).normal(0, 0.02, size=(2, 270, V))
    x = f32(x).reshape(2, 270, *nv)
    g["s2sh_x"] = x
    g["s2sh_c"] = signal_to_sh(DwiVolume(data=x, shells=3), op90).data
    # per-shell operators
    r30 = rand_dirs(rng, 30)
    g["pershell_dirs_b"] = r30
    ops = [make_fit_operator(d30, 4, 0.006), make_fit_operator(r30, 4, 0.006)]
    xp = f32(rng.normal(size=(1, 60, 3, 2, 2)) + 1.0)
    g["pershell_x"] = xp
    g["pershell_c"] = signal_to_sh(DwiVolume(data=xp, shells=2), ops).data
    # SH2Signal to the table and to 60 other directions
    c = f32(g["s2sh_c"])
    g["sh2s_c"] = c
    g["sh2s_y90"] = sh_to_signal(ShVolume(data=c, basis_spec=ShBasisSpec(8), shells=3), d90).data
    tgt = rand_dirs(rng, 60)
    g["sh2s_target60"] = tgt
    g["sh2s_y60"] = sh_to_signal(ShVolume(data=c, basis_spec=ShBasisSpec(8), shells=3), tgt).data
    # adjoints of the per-voxel maps (reference-anchored): dx = M^T dc, dc = B^T dy
    dc = f32(rng.normal(size=c.shape))
    g["s2sh_dc"] = dc
    Jm = jac(lambda e: signal_to_sh(DwiVolume(data=e, shells=1), op90).data, 90)  # (45, 90)
    g["s2sh_dx"] = np.einsum("rn,bsrv->bsnv", Jm, dc.reshape(2, 3, 45, -1)).reshape(2, 270, *nv)
    dy = f32(rng.normal(size=g["sh2s_y90"].shape))
    g["sh2s_dy"] = dy
    Jb = jac(lambda e: sh_to_signal(ShVolume(data=e, basis_spec=ShBasisSpec(8)), d90).data, 45)  # (90,45)
    g["sh2s_dc"] = np.einsum("nr,bsnv->bsrv", Jb, dy.reshape(2, 3, 90, -1)).reshape(2, 135, *nv)

    # ---- LSC forward + reference-anchored backward -------------------------------
    def lsc_case(tag, geo, order_in, si, so, c5, seed):
        r = np.random.default_rng(seed)
        K = geo.kernel_len
        w = f32(r.normal(size=(so, si, K)) / (si * K))
        b = f32(r.normal(size=so) * 0.1)
        g[f"{tag}_c"] = c5
        g[f"{tag}_w"] = w
        g[f"{tag}_b"] = b
        u = lsc_ref(c5, w, b, geo, order_in, si)
        g[f"{tag}_u"] = u
        gg = f32(np.random.default_rng(seed + 1).normal(size=u.shape))
        g[f"{tag}_g"] = gg
        rin = c5.shape[1] // si
        J = jac(lambda e: lsc_ref(e, w, np.zeros(so), geo, order_in, si), si * rin)
        nb = c5.shape[0]
        g[f"{tag}_dc"] = np.einsum("ji,bjv->biv", J, gg.reshape(nb, u.shape[1], -1)).reshape(c5.shape)
        dW = np.zeros_like(w)
        for o in range(so):
            for s in range(si):
                for k in range(K):
                    e = np.zeros_like(w)
                    e[o, s, k] = 1.0
                    dW[o, s, k] = np.sum(gg * lsc_ref(c5, e, np.zeros(so), geo, order_in, si))
        db = np.array([np.sum(gg * lsc_ref(np.zeros_like(c5), np.zeros_like(w), np.eye(so)[o], geo, order_in, si))
                       for o in range(so)])
        g[f"{tag}_dW"] = dW
        g[f"{tag}_db"] = db

    c3 = f32(g["s2sh_c"])
    lsc_case("lsc33", G["g90"], 8, 3, 3, c3, 1)
    lsc_case("lsc32", G["g90"], 8, 3, 2, c3, 3)           # S_in != S_out (never run by the reference tests)
    c1 = f32(rng.normal(size=(3, 45, 2, 3, 2)) * 0.2)
    c1[:, 0] = f32(2 * np.sqrt(np.pi))
    lsc_case("lsc11", G["g90"], 8, 1, 1, c1, 5)
    c4 = f32(rng.normal(size=(2, 15, 3, 1, 2)) * 0.3)
    lsc_case("lscr2", G["g30r2"], 4, 1, 1, c4, 7)         # two rings
    lsc_case("lsco42", G["g30o42"], 4, 1, 1, c4, 9)       # order_out != order_in

    # ---- fused chain: Signal2SH -> LSC 3->3 -> SH2Signal, fwd + bwd ---------------
    w = f32(np.random.default_rng(1).normal(size=(3, 3, 6)) / 18.0)
    b = f32(np.random.default_rng(1).normal(size=3) * 0.1)
    g["chain_w"] = w
    g["chain_b"] = b
    y = chain_ref(x, op90, G["g90"], w, b, d90, 8, 3)
    g["chain_y"] = y
    dyc = f32(np.random.default_rng(2).normal(size=y.shape))
    g["chain_dy"] = dyc
    J = jac(lambda e: chain_ref(e, op90, G["g90"], w, np.zeros(3), d90, 8, 3), 270)
    g["chain_dx"] = np.einsum("ji,bjv->biv", J, dyc.reshape(2, 270, -1)).reshape(x.shape)
    dW = np.zeros_like(w)
    for o in range(3):
        for s in range(3):
            for k in range(6):
                e = np.zeros_like(w)
                e[o, s, k] = 1.0
                dW[o, s, k] = np.sum(dyc * chain_ref(x, op90, G["g90"], e, np.zeros(3), d90, 8, 3))
    g["chain_dW"] = dW
    g["chain_db"] = np.array([np.sum(dyc * chain_ref(np.zeros_like(x), op90, G["g90"], np.zeros_like(w),
                                                       np.eye(3)[o], d90, 8, 3)) for o in range(3)])

    np.savez_compressed(OUT, **g)
    # the shipped direction tables as package data (directions.py:21-233 of the reference)
    os.makedirs(os.path.dirname(TABLES), exist_ok=True)
    np.savez_compressed(TABLES, **{f"dirs{n}": g[f"dirs{n}"] for n in (30, 60, 90)})
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
