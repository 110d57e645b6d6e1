"""float64 numpy restatement of sphdwi 0.1.0's hot path (the CPU oracle).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Reference paths below
are relative to /root/reference/pkg/src/sphdwi/.

Parity status: PINNED.  ``tests/test_oracle_golden.py`` checks every function
here against vectors produced by the real reference (``tests/golden/
make_golden.py``) and against the reference tests' own known-answer values.

The reference has no backward pass.  The adjoints
below are restated per stage from the reference's forward structure (resample
-> ring reduce -> refit, _kernels.py:91-104 + lsc.py:197), not from the folded
operator the CUDA path uses, and are pinned by reference-anchored Jacobians
(the forward is exactly linear, so J^T dy is recoverable from reference calls
on basis vectors; see make_golden.py).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

SH_C0 = 0.28209479177387814          # shcore.py:28
TWO_SQRT_PI = 2.0 * np.sqrt(np.pi)
COND_LIMIT = 1e12                    # fitting.py:30
BLOCK = 1024                         # fitting.py:152


class OracleError(ValueError):
    """Raised where the reference raises ShapeError / IllPosedFitError / ValueError."""


# --------------------------------------------------------------------------- shcore
def coeff_count(order: int) -> int:
    """shcore.py:33-41 -- R = (L+1)(L+2)/2 for even L >= 0."""
    if order < 0 or order % 2:
        raise OracleError(f"SH order must be even and >= 0, got {order}")
    return (order + 1) * (order + 2) // 2


def degrees(order: int) -> np.ndarray:
    """shcore.py:80-86 -- degree l of every packed index j = l(l+1)/2 + m."""
    coeff_count(order)
    return np.concatenate([np.full(2 * l + 1, l) for l in range(0, order + 1, 2)]).astype(np.int64)


def unit(dirs) -> np.ndarray:
    """shcore.py:92-109 -- validate and normalise (N,3) directions."""
    a = np.atleast_2d(np.asarray(dirs, dtype=np.float64))
    if a.ndim != 2 or a.shape[1] != 3 or a.shape[0] == 0 or not np.isfinite(a).all():
        raise OracleError(f"bad direction array {a.shape}")
    n = np.linalg.norm(a, axis=1)
    if np.any(n <= 1e-12):
        raise OracleError("zero direction vector")
    return a / n[:, None]


def eval_basis(dirs, order: int) -> np.ndarray:
    """shcore.py:112-166 -- real even-order SH basis, (N, R).

    Normalised associated-Legendre recurrence in l (Condon-Shortley folded in,
    :132-145), Chebyshev recurrences for cos/sin(m phi) (:147-156), poles map to
    cos phi = 1, sin phi = 0 (:123-128); sqrt2*N*cos for m<0, sqrt2*N*sin for
    m>0 (:158-165).
    """
    R = coeff_count(order)
    u = unit(dirs)
    x, y, z = u[:, 0], u[:, 1], u[:, 2]
    rho = np.hypot(x, y)
    pos = rho > 0.0
    cph = np.where(pos, x / np.where(pos, rho, 1.0), 1.0)
    sph = np.where(pos, y / np.where(pos, rho, 1.0), 0.0)
    L = order
    P = {}
    P[(0, 0)] = np.full(u.shape[0], SH_C0)
    for m in range(1, L + 1):
        P[(m, m)] = -np.sqrt((2.0 * m + 1.0) / (2.0 * m)) * rho * P[(m - 1, m - 1)]
    for m in range(0, L + 1):
        if m + 1 <= L:
            P[(m + 1, m)] = np.sqrt(2.0 * m + 3.0) * z * P[(m, m)]
        for l in range(m + 2, L + 1):
            a = np.sqrt((4.0 * l * l - 1.0) / (l * l - m * m))
            b = np.sqrt(((2.0 * l + 1.0) * ((l - 1.0) ** 2 - m * m)) / ((2.0 * l - 3.0) * (l * l - m * m)))
            P[(l, m)] = a * z * P[(l - 1, m)] - b * P[(l - 2, m)]
    cm = [np.ones_like(x), cph]
    sm = [np.zeros_like(x), sph]
    for m in range(2, L + 1):
        cm.append(2.0 * cph * cm[m - 1] - cm[m - 2])
        sm.append(2.0 * cph * sm[m - 1] - sm[m - 2])
    out = np.empty((u.shape[0], R))
    r2 = np.sqrt(2.0)
    for l in range(0, L + 1, 2):
        c = l * (l + 1) // 2
        out[:, c] = P[(l, 0)]
        for m in range(1, l + 1):
            out[:, c - m] = r2 * P[(l, m)] * cm[m]
            out[:, c + m] = r2 * P[(l, m)] * sm[m]
    return out


def lb_diag(order: int) -> np.ndarray:
    """shcore.py:169-172 -- l^2 (l+1)^2."""
    l = degrees(order).astype(np.float64)
    return (l * (l + 1.0)) ** 2


def tangent_frame(u):
    """shcore.py:175-186 -- e1 = normalize(ref x u), ref=+z unless |u_z|>0.9 (+x)."""
    uu = unit(u)[0]
    ref = np.array([0.0, 0.0, 1.0]) if abs(uu[2]) <= 0.9 else np.array([1.0, 0.0, 0.0])
    e1 = np.cross(ref, uu)
    e1 = e1 / np.linalg.norm(e1)
    return e1, np.cross(uu, e1)


def ring(u, alpha: float, n: int) -> np.ndarray:
    """shcore.py:189-206 -- n points at angle alpha around u, phase 0 along e1."""
    if not (0.0 < alpha < np.pi / 2.0) or n < 1:
        raise OracleError("bad ring")
    uu = unit(u)[0]
    e1, e2 = tangent_frame(uu)
    az = 2.0 * np.pi * np.arange(n) / n
    pts = np.cos(alpha) * uu[None] + np.sin(alpha) * (np.cos(az)[:, None] * e1[None] + np.sin(az)[:, None] * e2[None])
    return pts / np.linalg.norm(pts, axis=1, keepdims=True)


# --------------------------------------------------------------------------- fitting
def fit_operator(dirs, order: int, lam: float = 0.0):
    """fitting.py:108-149 -- M = (B^T B + lam diag(LB))^-1 B^T by Cholesky.

    Returns (M (R,N), B (N,R), cond).  Same rejection rules: lam < 0,
    lam == 0 with N < R, cond > 1e12, not positive definite.
    """
    d = unit(dirs)
    if lam < 0:
        raise OracleError("lambda < 0")
    R = coeff_count(order)
    if lam == 0.0 and d.shape[0] < R:
        raise OracleError("underdetermined")
    B = eval_basis(d, order)
    A = B.T @ B + lam * np.diag(lb_diag(order))
    cond = float(np.linalg.cond(A))
    if not np.isfinite(cond) or cond > COND_LIMIT:
        raise OracleError("ill-conditioned")
    M = scipy.linalg.cho_solve(scipy.linalg.cho_factor(A), B.T)
    return np.ascontiguousarray(M), B, cond


def apply_channel_matrix(W: np.ndarray, stacked: np.ndarray) -> np.ndarray:
    """fitting.py:155-188 -- out[b,s] = W @ stacked[b,s] in 1024-voxel zero-padded blocks."""
    nb, ns, cin, nv = stacked.shape
    out = np.empty((nb, ns, W.shape[0], nv))
    for b in range(nb):
        for s in range(ns):
            for lo in range(0, nv, BLOCK):
                hi = min(nv, lo + BLOCK)
                buf = np.zeros((cin, BLOCK))
                buf[:, : hi - lo] = stacked[b, s, :, lo:hi]
                out[b, s, :, lo:hi] = (W @ buf)[:, : hi - lo]
    return out


def signal_to_sh(x5: np.ndarray, M, shells: int) -> np.ndarray:
    """fitting.py:206-236 -- per-shell fit; M is one (R,N) matrix or a list per shell."""
    Ms = [M] if isinstance(M, np.ndarray) else list(M)
    if len(Ms) == 1:
        Ms = Ms * shells
    R, N = Ms[0].shape
    B_, C = x5.shape[:2]
    if C != shells * N:
        raise OracleError("channel mismatch")
    grid = x5.shape[2:]
    st = np.asarray(x5, np.float64).reshape(B_, shells, N, -1)
    out = np.concatenate([apply_channel_matrix(Ms[s], st[:, s : s + 1]) for s in range(shells)], axis=1)
    return out.reshape(B_, shells * R, *grid)


def sh_to_signal(c5: np.ndarray, Bt: np.ndarray, shells: int) -> np.ndarray:
    """fitting.py:239-250 -- y[b,s] = B' c[b,s] at target directions."""
    N, R = Bt.shape
    B_ = c5.shape[0]
    grid = c5.shape[2:]
    st = np.asarray(c5, np.float64).reshape(B_, shells, R, -1)
    return apply_channel_matrix(Bt, st).reshape(B_, shells * N, *grid)


# --------------------------------------------------------------------------- LSC
def lsc_geometry(origins, sizes, alpha: float, order_in: int, order_out: int, lam: float = 0.0):
    """lsc.py:87-135 -- rings at r*alpha, origin-major rows [origin, ring1.., ring2..].

    Returns dict(resample (m*K, R_in), refit (R_out, m), K, m, dirs (m*K,3)).
    """
    o = unit(origins)
    sizes = tuple(int(s) for s in sizes)
    if not sizes or any(s < 1 for s in sizes):
        raise OracleError("kernel sizes")
    if alpha <= 0.0 or alpha * len(sizes) >= np.pi / 2.0:
        raise OracleError("hemisphere")
    m = o.shape[0]
    K = 1 + sum(sizes)
    rings = [np.stack([ring(u, r * alpha, n) for u in o]) for r, n in enumerate(sizes, start=1)]
    dirs = np.empty((m * K, 3))
    for i in range(m):
        dirs[i * K : (i + 1) * K] = np.concatenate([o[i : i + 1]] + [rg[i] for rg in rings])
    F, _, _ = fit_operator(o, order_out, lam)
    return {"resample": eval_basis(dirs, order_in), "refit": F, "K": K, "m": m, "dirs": dirs}


def lsc_combine(resample, w, bias, coeffs) -> np.ndarray:
    """_kernels.py:91-104 -- u[o,i,v] = bias[o] + sum_{s,k} w[o,s,k] (Rs[iK+k] . c[s,:,v])."""
    so, si, K = w.shape
    m = resample.shape[0] // K
    V = coeffs.shape[-1]
    out = np.empty((so, m, V))
    chunk = max(1, int(4_000_000 // max(1, m * K * si)))               # _kernels.py:97
    for lo in range(0, V, chunk):
        hi = min(V, lo + chunk)
        S = np.matmul(resample, coeffs[:, :, lo:hi]).reshape(si, m, K, hi - lo)
        out[:, :, lo:hi] = np.einsum("osk,smkv->omv", w, S)
    return out + bias[:, None, None]


def lsc_forward(c5: np.ndarray, w, bias, geom) -> np.ndarray:
    """lsc.py:158-199 -- combine per subject, then refit every output shell."""
    w = np.asarray(w, np.float64)
    bias = np.asarray(bias, np.float64)
    so, si, K = w.shape
    if K != geom["K"]:
        raise OracleError("K mismatch")
    Rin = geom["resample"].shape[1]
    if c5.shape[1] != si * Rin:
        raise OracleError("shell mismatch")
    B_ = c5.shape[0]
    grid = c5.shape[2:]
    F = geom["refit"]
    st = np.asarray(c5, np.float64).reshape(B_, si, Rin, -1)
    out = np.empty((B_, so * F.shape[0], st.shape[-1]))
    for b in range(B_):
        u = lsc_combine(geom["resample"], w, bias, st[b])
        out[b] = apply_channel_matrix(F, u[None])[0].reshape(so * F.shape[0], -1)
    return out.reshape(B_, so * F.shape[0], *grid)


# --------------------------------------------------------------------------- adjoints
def signal_to_sh_adjoint(dc5, M, shells: int) -> np.ndarray:
    """d(signal_to_sh)^T: dx[b,s] = M_s^T dc[b,s]."""
    Ms = [M] if isinstance(M, np.ndarray) else list(M)
    if len(Ms) == 1:
        Ms = Ms * shells
    R, N = Ms[0].shape
    B_ = dc5.shape[0]
    grid = dc5.shape[2:]
    st = np.asarray(dc5, np.float64).reshape(B_, shells, R, -1)
    out = np.stack([np.matmul(Ms[s].T, st[:, s]) for s in range(shells)], axis=1)
    return out.reshape(B_, shells * N, *grid)


def sh_to_signal_adjoint(dy5, Bt, shells: int) -> np.ndarray:
    """d(sh_to_signal)^T: dc[b,s] = B'^T dy[b,s]."""
    N, R = Bt.shape
    B_ = dy5.shape[0]
    grid = dy5.shape[2:]
    st = np.asarray(dy5, np.float64).reshape(B_, shells, N, -1)
    return np.matmul(Bt.T, st).reshape(B_, shells * R, *grid)


def lsc_backward(c5, g5, w, geom):
    """Adjoint of lsc_forward, stage by stage (refit^T, ring-reduce^T, resample^T).

    Returns (dc_in like c5, dW (S_out,S_in,K), db (S_out,)).
    """
    w = np.asarray(w, np.float64)
    so, si, K = w.shape
    Rs, F = geom["resample"], geom["refit"]
    Rin, Rout, m = Rs.shape[1], F.shape[0], geom["m"]
    B_ = c5.shape[0]
    grid = c5.shape[2:]
    c = np.asarray(c5, np.float64).reshape(B_, si, Rin, -1)
    g = np.asarray(g5, np.float64).reshape(B_, so, Rout, -1)
    dc = np.empty_like(c)
    dW = np.zeros((so, si, K))
    db = np.zeros(so)
    chunk = max(1, int(4_000_000 // max(1, m * K * si)))                # same blocking as _kernels.py:97
    for b in range(B_):
        for lo in range(0, c.shape[-1], chunk):
            hi = min(c.shape[-1], lo + chunk)
            V = hi - lo
            ubar = np.matmul(F.T, g[b][:, :, lo:hi])                    # refit^T   (so, m, V)
            S = np.matmul(Rs, c[b][:, :, lo:hi]).reshape(si, m, K, V)   # resample  (si, m, K, V)
            Sbar = np.empty((si, m, K, V))
            u2 = ubar.reshape(so, m * V)
            for k in range(K):                                          # ring reduce^T, per kernel point
                Sk = np.ascontiguousarray(S[:, :, k, :]).reshape(si, m * V)
                dW[:, :, k] += u2 @ Sk.T
                Sbar[:, :, k, :] = (w[:, :, k].T @ u2).reshape(si, m, V)
            db += ubar.sum(axis=(1, 2))
            dc[b][:, :, lo:hi] = np.matmul(Rs.T, Sbar.reshape(si, m * K, V))   # resample^T
    return dc.reshape(B_, si * Rin, *grid), dW, db


# --------------------------------------------------------------------------- the fused chain
def chain_forward(x5, M, geom, w, bias, Bt, shells_in: int):
    """Signal2SH -> LSC -> SH2Signal (SURVEY.md §3 stack 4, in-memory layers)."""
    c = signal_to_sh(x5, M, shells_in)
    u = lsc_forward(c, w, bias, geom)
    return sh_to_signal(u, Bt, np.asarray(w).shape[0])


def chain_backward(x5, dy5, M, geom, w, Bt, shells_in: int):
    """(dx, dW, db) of <chain_forward(x), dy>."""
    so = np.asarray(w).shape[0]
    c = signal_to_sh(x5, M, shells_in)
    g = sh_to_signal_adjoint(dy5, Bt, so)
    dc, dW, db = lsc_backward(c, g, w, geom)
    return signal_to_sh_adjoint(dc, M, shells_in), dW, db


# --------------------------------------------------------------------------- synthetic inputs
def bandlimited_coeffs(rng: np.random.Generator, order: int, nvox: int) -> np.ndarray:
    """phantom.py:77-88 -- c0 = 2 sqrt(pi), others U(-1,1) * 0.9/(1 + l(l+1)/4)."""
    l = degrees(order).astype(np.float64)
    c = rng.uniform(-1.0, 1.0, size=(coeff_count(order), nvox)) * (0.9 / (1.0 + l * (l + 1.0) / 4.0))[:, None]
    c[0] = TWO_SQRT_PI
    return c


def rel_err(got, ref) -> float:
    """Normwise max relative error max|got-ref| / max|ref|."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = float(np.max(np.abs(ref))) if ref.size else 0.0
    num = float(np.max(np.abs(got - ref))) if ref.size else 0.0
    return num / den if den > 0 else num
