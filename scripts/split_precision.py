"""Emulate the chain kernel's split-operand tensor-core arithmetic on the CPU (design probe, not a test).

Every fp32 operand a is written as a sum of low-precision terms (bf16 or fp16); the MMA forms the products of
the term pairs (i, j) with i + j < P exactly and accumulates them in fp32.  Compares, against the fp64
oracle chain, the schemes the kernel can use: bf16 x3 (6 MMAs / K-step), bf16 x2 (3 MMAs), fp16 x2 (3 MMAs,
activations scaled by a power of two `scale`).
usage: python scripts/split_precision.py [nvox]
"""
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
from oracle import port  # noqa: E402
from paper_1808_01517_b200.directions import unit_sphere_directions  # noqa: E402


def to_bf16(a):
    a = np.asarray(a, np.float32)
    b = a.view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def to_fp16(a):
    return np.asarray(a, np.float32).astype(np.float16).astype(np.float32)


def split(a, kind, parts):
    f = to_bf16 if kind == "bf16" else to_fp16
    out, r = [], np.asarray(a, np.float32)
    for _ in range(parts):
        t = f(r)
        out.append(t)
        r = (r - t).astype(np.float32)
    return out


def mm(W, X, kind, parts, scale=1.0):
    """W (n,k) fp32 weights, X (k,v) fp32 activations -> fp32 W @ X with split terms."""
    Ws = split(W, kind, parts)
    Xs = split(X * np.float32(scale), kind, parts)
    acc = np.zeros((W.shape[0], X.shape[1]), np.float32)
    for i in range(parts):
        for j in range(parts):
            if i + j < parts:
                acc += (Ws[j].astype(np.float32) @ Xs[i].astype(np.float32)).astype(np.float32)
    return acc / np.float32(scale)


def main():
    V = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    dirs = unit_sphere_directions(90)
    M, _, _ = port.fit_operator(dirs, 8, 0.006)
    geom = port.lsc_geometry(dirs, [5], np.pi / 5, 8, 8, 0.006)
    S, K = 3, geom["K"]
    w = np.random.default_rng(1).normal(size=(S, S, K)) / (S * K)
    bias = np.random.default_rng(1).normal(size=S) * 0.1
    Bt = port.eval_basis(dirs, 8)
    F, Rs = geom["refit"], geom["resample"]
    P = np.stack([F @ Rs[k::K] for k in range(K)])
    L = np.einsum("osk,kab->oasb", w, P).reshape(S * 45, S * 45)
    beta = F @ np.ones(F.shape[1])
    rng = np.random.default_rng(0)
    x = np.concatenate([Bt @ port.bandlimited_coeffs(rng, 8, V) + 0.02 * rng.normal(size=(90, V)) for _ in range(S)])
    x32 = x.astype(np.float32)
    Mbd = np.kron(np.eye(S), M)
    Bbd = np.kron(np.eye(S), Bt)
    ub = np.kron(bias, beta)[:, None]
    ref = Bbd @ (L @ (Mbd @ x32.astype(np.float64)) + ub)
    dy = rng.normal(size=ref.shape).astype(np.float32)
    refb = Mbd.T @ (L.T @ (Bbd.T @ dy.astype(np.float64)))
    for kind, parts in (("bf16", 3), ("bf16", 2), ("fp16", 2)):
        for scale in ((1.0,) if kind == "bf16" else (1.0, 2.0 ** 6, 2.0 ** -20)):
            W1, W2, W3 = (np.float32(Mbd), np.float32(L), np.float32(Bbd))
            c = mm(W1, x32, kind, parts, scale)
            u = mm(W2, c, kind, parts, scale) + np.float32(ub)
            y = mm(W3, u, kind, parts, scale)
            g = mm(W3.T.copy(), dy * np.float32(2.0 ** -30 if scale == 2.0 ** -20 else 1), kind, parts,
                   scale * (2.0 ** 30 if scale == 2.0 ** -20 else 1))
            d = mm(W1.T.copy(), mm(W2.T.copy(), g, kind, parts, scale), kind, parts, scale)
            if scale == 2.0 ** -20:
                d = d * np.float32(2.0 ** 30)
            print(f"{kind} x{parts} scale 2^{int(np.log2(scale)):+d}: fwd rel {port.rel_err(y, ref):.2e}  "
                  f"adj rel {port.rel_err(d, refb):.2e}")


if __name__ == "__main__":
    main()
