"""Host-side float64 builders: SH basis, regularised fit operators, LSC geometry.

Built once per gradient table on the host (as the reference does) and uploaded
to the device as float32 constants.  Conventions follow the reference
(/root/reference/pkg/src/sphdwi/shcore.py:1-20):

* even degrees only, R = (L+1)(L+2)/2, packed index j = l(l+1)/2 + m;
* real basis sqrt2*N*cos(m phi) for m < 0, N for m = 0, sqrt2*N*sin(m phi) for m > 0,
  with the fully normalised associated Legendre N_l^|m| (Condon-Shortley folded in);
* theta from +z, phi from +x; at the poles cos phi = 1, sin phi = 0.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import scipy.linalg

from .errors import IllPosedFitError, ShapeError

SH_C0 = 0.28209479177387814   # Y_0^0 (shcore.py:28)
COND_LIMIT = 1e12             # fitting.py:30
TWO_SQRT_PI = 2.0 * np.sqrt(np.pi)


# ----------------------------------------------------------------------------- packing
def _check_order(order: int) -> None:
    if int(order) != order or order < 0 or order % 2:
        raise ValueError(f"SH order must be even and >= 0, got {order}")


def coeff_count(order: int) -> int:
    """R for max degree `order` (shcore.py:33-41)."""
    _check_order(order)
    return (order + 1) * (order + 2) // 2


def sh_index(l: int, m: int) -> int:
    """j = l(l+1)/2 + m (shcore.py:62-68)."""
    if l < 0 or l % 2:
        raise ValueError(f"degree must be even and >= 0, got l={l}")
    if abs(m) > l:
        raise ValueError(f"order m must satisfy |m| <= l, got l={l}, m={m}")
    return l * (l + 1) // 2 + m


def sh_degree_order(j: int) -> tuple[int, int]:
    """Inverse of sh_index (shcore.py:71-79)."""
    if j < 0:
        raise ValueError(f"coefficient index must be >= 0, got {j}")
    l = 0
    while l * (l + 1) // 2 + l < j:
        l += 2
    return l, j - l * (l + 1) // 2


def basis_degrees(order: int) -> np.ndarray:
    """Degree of every packed coefficient (shcore.py:80-86)."""
    _check_order(order)
    return np.repeat(np.arange(0, order + 1, 2), np.arange(0, order + 1, 2) * 2 + 1).astype(np.int64)


@dataclass(frozen=True)
class ShBasisSpec:
    """Shape descriptor of an even-order real SH basis (shcore.py:44-59)."""

    order: int

    def __post_init__(self) -> None:
        _check_order(self.order)

    @property
    def coeff_count(self) -> int:
        return coeff_count(self.order)

    def degrees(self) -> np.ndarray:
        return basis_degrees(self.order)


# ----------------------------------------------------------------------------- directions / basis
def as_unit_directions(dirs) -> np.ndarray:
    """(N,3) unit rows; rejects empty, non-finite and zero rows (shcore.py:92-109)."""
    arr = np.atleast_2d(np.asarray(dirs, dtype=np.float64))
    if arr.ndim != 2 or arr.shape[1] != 3:
        raise ValueError(f"directions must have shape (N, 3), got {arr.shape}")
    if arr.shape[0] == 0:
        raise ValueError("direction list is empty")
    if not np.isfinite(arr).all():
        raise ValueError("directions contain non-finite values")
    norms = np.linalg.norm(arr, axis=1)
    bad = np.flatnonzero(norms <= 1e-12)
    if bad.size:
        raise ValueError(f"zero direction vector at row {int(bad[0])}")
    return arr / norms[:, None]


def eval_basis(dirs, order: int) -> np.ndarray:
    """B[i, j] = Y_j(u_i), shape (N, R) (shcore.py:112-166).

    Legendre: sectoral seed N_m^m = -sqrt((2m+1)/(2m)) rho N_{m-1}^{m-1}, first
    step N_{m+1}^m = sqrt(2m+3) z N_m^m, then the three-term recurrence in l.
    Azimuth: Chebyshev recurrences on (cos phi, sin phi).
    """
    _check_order(order)
    u = as_unit_directions(dirs)
    n, L = u.shape[0], order
    x, y, z = u.T
    rho = np.hypot(x, y)
    nz = rho > 0.0
    den = np.where(nz, rho, 1.0)
    cphi = np.where(nz, x / den, 1.0)
    sphi = np.where(nz, y / den, 0.0)

    P = np.zeros((L + 1, L + 1, n))          # P[l, m]
    P[0, 0] = SH_C0
    for m in range(1, L + 1):
        P[m, m] = -np.sqrt((2.0 * m + 1.0) / (2.0 * m)) * rho * P[m - 1, m - 1]
    for m in range(L + 1):
        if m < L:
            P[m + 1, m] = np.sqrt(2.0 * m + 3.0) * z * P[m, m]
        for l in range(m + 2, L + 1):
            ll, mm = float(l * l), float(m * m)
            a = np.sqrt((4.0 * ll - 1.0) / (ll - mm))
            b = np.sqrt(((2.0 * l + 1.0) * ((l - 1.0) ** 2 - mm)) / ((2.0 * l - 3.0) * (ll - mm)))
            P[l, m] = a * z * P[l - 1, m] - b * P[l - 2, m]

    C = np.empty((L + 1, n))
    S = np.empty((L + 1, n))
    C[0], S[0] = 1.0, 0.0
    if L >= 1:
        C[1], S[1] = cphi, sphi
    for m in range(2, L + 1):
        C[m] = 2.0 * cphi * C[m - 1] - C[m - 2]
        S[m] = 2.0 * cphi * S[m - 1] - S[m - 2]

    out = np.empty((n, coeff_count(L)))
    r2 = np.sqrt(2.0)
    for l in range(0, L + 1, 2):
        c = l * (l + 1) // 2
        out[:, c] = P[l, 0]
        ms = np.arange(1, l + 1)
        out[:, c - ms] = (r2 * P[l, 1 : l + 1] * C[1 : l + 1]).T
        out[:, c + ms] = (r2 * P[l, 1 : l + 1] * S[1 : l + 1]).T
    return out


def laplace_beltrami_diag(order: int) -> np.ndarray:
    """l^2 (l+1)^2 per coefficient (shcore.py:169-172)."""
    l = basis_degrees(order).astype(np.float64)
    return (l * (l + 1.0)) ** 2


def tangent_basis(u) -> tuple[np.ndarray, np.ndarray]:
    """Right-handed (e1, e2) at u; reference axis +z, +x when |u_z| > 0.9 (shcore.py:175-186)."""
    uu = as_unit_directions(u)[0]
    ref = np.array([0.0, 0.0, 1.0]) if abs(uu[2]) <= 0.9 else np.array([1.0, 0.0, 0.0])
    e1 = np.cross(ref, uu)
    e1 /= np.linalg.norm(e1)
    return e1, np.cross(uu, e1)


def ring_directions(u, alpha: float, n: int) -> np.ndarray:
    """n points at angle alpha around u, phase 0 along e1, renormalised (shcore.py:189-206)."""
    if not (0.0 < alpha < np.pi / 2.0):
        raise ValueError(f"angular distance must lie in (0, pi/2), got {alpha}")
    if n < 1:
        raise ValueError(f"ring point count must be >= 1, got {n}")
    uu = as_unit_directions(u)[0]
    e1, e2 = tangent_basis(uu)
    az = 2.0 * np.pi * np.arange(n) / n
    pts = np.cos(alpha) * uu[None, :] + np.sin(alpha) * (np.cos(az)[:, None] * e1[None, :] + np.sin(az)[:, None] * e2[None, :])
    return pts / np.linalg.norm(pts, axis=1, keepdims=True)


def degree_energies(coeffs, order: int, axis: int = 0) -> np.ndarray:
    """Sum of squared coefficients per even degree (shcore.py:209-226)."""
    arr = np.moveaxis(np.asarray(coeffs, dtype=np.float64), axis, 0)
    if arr.shape[0] != coeff_count(order):
        raise ValueError(f"expected {coeff_count(order)} coefficients along axis {axis}, got {arr.shape[0]}")
    degs = basis_degrees(order)
    out = np.stack([np.sum(arr[degs == l] ** 2, axis=0) for l in range(0, order + 1, 2)], axis=0)
    return np.moveaxis(out, 0, axis)


def high_degree_energy_fraction(coeffs, order: int, axis: int = 0, min_degree: int = 2) -> np.ndarray:
    """Energy fraction in degrees >= min_degree (shcore.py:229-237)."""
    en = np.moveaxis(degree_energies(coeffs, order, axis=axis), axis, 0)
    lv = np.arange(0, order + 1, 2)
    tot = en.sum(axis=0)
    hi = en[lv >= min_degree].sum(axis=0)
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(tot > 0.0, hi / tot, 0.0)


# ----------------------------------------------------------------------------- fit operator
@dataclass(frozen=True)
class FitOperator:
    """Sample -> coefficient map M = (B^T B + lambda diag(LB))^-1 B^T (fitting.py:92-105)."""

    basis_spec: ShBasisSpec
    gradients: np.ndarray       # (N, 3)
    lb_lambda: float
    basis_matrix: np.ndarray    # (N, R)
    fit_matrix: np.ndarray      # (R, N)
    cond: float

    @property
    def n_gradients(self) -> int:
        return int(self.gradients.shape[0])


def make_fit_operator(gradients, order: int, lb_lambda: float = 0.0) -> FitOperator:
    """Regularised least-squares operator via Cholesky (fitting.py:108-149).

    Raises ValueError for lambda < 0 and IllPosedFitError for lambda == 0 with
    N < R, for cond > 1e12 and for a normal matrix that is not positive definite.
    """
    dirs = as_unit_directions(gradients)
    if lb_lambda < 0:
        raise ValueError(f"regularization weight must be >= 0, got {lb_lambda}")
    n, r = dirs.shape[0], coeff_count(order)
    if lb_lambda == 0.0 and n < r:
        raise IllPosedFitError(f"unregularized fit needs at least R = {r} directions, got N = {n} (cond = inf)")
    B = eval_basis(dirs, order)
    A = B.T @ B + lb_lambda * np.diag(laplace_beltrami_diag(order))
    cond = float(np.linalg.cond(A))
    if not np.isfinite(cond) or cond > COND_LIMIT:
        raise IllPosedFitError(f"fit system is numerically rank deficient (N = {n}, R = {r}, cond = {cond:.3e})")
    try:
        chol = scipy.linalg.cho_factor(A)
    except scipy.linalg.LinAlgError as exc:
        raise IllPosedFitError(f"normal matrix is not positive definite (N = {n}, R = {r}, cond = {cond:.3e})") from exc
    M = np.ascontiguousarray(scipy.linalg.cho_solve(chol, B.T))
    for a in (dirs, B, M):
        a.setflags(write=False)
    return FitOperator(ShBasisSpec(order), dirs, float(lb_lambda), B, M, cond)


# ----------------------------------------------------------------------------- LSC
@dataclass(frozen=True)
class LscKernel:
    """Ring-kernel weights (shells_out, shells_in, K) and bias (shells_out,) (lsc.py:30-59)."""

    weights: np.ndarray
    bias: np.ndarray

    def __post_init__(self) -> None:
        w = np.ascontiguousarray(np.asarray(self.weights, dtype=np.float64))
        b = np.ascontiguousarray(np.asarray(self.bias, dtype=np.float64))
        if w.ndim != 3:
            raise ShapeError(f"kernel weights must be (shells_out, shells_in, K), got {w.shape}")
        if b.shape != (w.shape[0],):
            raise ShapeError(f"bias must have one entry per output shell, got {b.shape}")
        if not (np.isfinite(w).all() and np.isfinite(b).all()):
            raise ShapeError("kernel contains non-finite entries")
        object.__setattr__(self, "weights", w)
        object.__setattr__(self, "bias", b)

    @property
    def shells_out(self) -> int:
        return self.weights.shape[0]

    @property
    def shells_in(self) -> int:
        return self.weights.shape[1]

    @property
    def kernel_len(self) -> int:
        return self.weights.shape[2]


@dataclass(frozen=True)
class LscGeometry:
    """Ring resampling + refit for one origin set (lsc.py:62-84), plus the folded operator.

    fold (K, R_out, R_in) = refit . resample[k::K] and beta = refit . 1 are the
    per-geometry constants the CUDA path uses.
    """

    origins: np.ndarray
    alpha: float
    kernel_sizes: tuple
    order_in: int
    rings: tuple
    resample_matrix: np.ndarray     # (m*K, R_in)
    refit: FitOperator
    fold: np.ndarray = field(repr=False, default=None)
    beta: np.ndarray = field(repr=False, default=None)

    @property
    def m(self) -> int:
        return int(self.origins.shape[0])

    @property
    def kernel_len(self) -> int:
        return 1 + sum(self.kernel_sizes)

    @property
    def order_out(self) -> int:
        return self.refit.basis_spec.order


def _check_sizes(kernel_sizes) -> tuple:
    sizes = tuple(int(s) for s in kernel_sizes)
    if not sizes or any(s < 1 for s in sizes):
        raise ValueError(f"kernel_sizes must be non-empty positive integers, got {kernel_sizes}")
    return sizes


def build_lsc_geometry(gradients, kernel_sizes, alpha: float, order_in: int, order_out: int,
                       lb_lambda: float = 0.0) -> LscGeometry:
    """Rings at r*alpha, origin-major rows [origin, ring-1.., ring-2..] (lsc.py:87-135)."""
    origins = as_unit_directions(gradients)
    sizes = _check_sizes(kernel_sizes)
    if alpha <= 0.0 or alpha * len(sizes) >= np.pi / 2.0:
        raise ValueError(f"rings must stay inside the hemisphere: need 0 < alpha and alpha * {len(sizes)} < pi/2, "
                         f"got alpha = {alpha}")
    _check_order(order_in)
    m, K = origins.shape[0], 1 + sum(sizes)
    rings = tuple(np.stack([ring_directions(u, r * alpha, n) for u in origins]) for r, n in enumerate(sizes, start=1))
    blocks = [origins[:, None, :]] + [rg for rg in rings]
    dirs = np.concatenate(blocks, axis=1).reshape(m * K, 3)
    resample = eval_basis(dirs, order_in)
    refit = make_fit_operator(origins, order_out, lb_lambda)
    F = refit.fit_matrix
    fold = np.ascontiguousarray(np.einsum("ri,ikt->krt", F, resample.reshape(m, K, -1)))
    beta = F.sum(axis=1)
    for a in (resample, fold, beta):
        a.setflags(write=False)
    return LscGeometry(origins, float(alpha), sizes, int(order_in), rings, resample, refit, fold, beta)


def make_moving_average_kernel(kernel_sizes, shells_in: int = 1, shells_out: int = 1) -> LscKernel:
    """Every weight 1/(shells_in*K), zero bias (lsc.py:138-145)."""
    K = 1 + sum(_check_sizes(kernel_sizes))
    return LscKernel(np.full((shells_out, shells_in, K), 1.0 / (shells_in * K)), np.zeros(shells_out))


def make_identity_kernel(kernel_sizes, shells: int = 1) -> LscKernel:
    """w[s, s, 0] = 1: keeps each shell's origin sample (lsc.py:148-155)."""
    K = 1 + sum(int(s) for s in kernel_sizes)
    w = np.zeros((shells, shells, K))
    w[np.arange(shells), np.arange(shells), 0] = 1.0
    return LscKernel(w, np.zeros(shells))


def per_shell_operators(op, shells: int) -> list:
    """Shared or per-shell operators with a common order and N (fitting.py:191-203)."""
    ops = [op] if isinstance(op, FitOperator) else list(op)
    if len(ops) == 1:
        ops = ops * shells
    if len(ops) != shells:
        raise ShapeError(f"got {len(ops)} fit operators for {shells} shells")
    for other in ops[1:]:
        if other.basis_spec.order != ops[0].basis_spec.order:
            raise ShapeError("per-shell fit operators must share one SH order")
        if other.n_gradients != ops[0].n_gradients:
            raise ShapeError("per-shell fit operators must share one gradient count")
    return ops


def seq_or_single(gradients) -> tuple[list, bool]:
    """(list of (N,3) tables, per_shell?) from an (N,3) or (S,N,3) gradient argument."""
    arr = np.asarray(gradients, dtype=np.float64)
    if arr.ndim == 3:
        return [arr[s] for s in range(arr.shape[0])], True
    return [arr], False


__all__: Sequence[str] = [
    "SH_C0", "TWO_SQRT_PI", "ShBasisSpec", "coeff_count", "sh_index", "sh_degree_order", "basis_degrees",
    "as_unit_directions", "eval_basis", "laplace_beltrami_diag", "tangent_basis", "ring_directions",
    "degree_energies", "high_degree_energy_fraction", "FitOperator", "make_fit_operator", "LscKernel",
    "LscGeometry", "build_lsc_geometry", "make_moving_average_kernel", "make_identity_kernel",
]
