"""Drop-in functional API mirroring sphdwi's operator surface, on the GPU.

Same names, argument meaning and errors as the reference:

* signal_to_sh(vol, op, threads=1) -> ShVolume           (fitting.py:206-236)
* sh_to_signal(sh, gradients, threads=1) -> DwiVolume    (fitting.py:239-250)
* lsc_forward(sh_in, kernel, geom, threads=1, backend=None) -> ShVolume  (lsc.py:158-199)
* apply_channel_matrix(matrix, stacked, threads=1, out=None)            (fitting.py:155-188)
* lsc_combine(resample, weights, bias, coeffs, backend=None)            (_kernels.py:187-206)

ShVolume / DwiVolume hold an fp32 CUDA tensor instead of a float64 numpy array.
`threads` and `backend` are accepted for signature compatibility; the single
implementation is the sm_100a kernel set, so they do not select anything.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import ops
from .errors import KernelMismatchError, ShapeError
from .geometry import (
    FitOperator,
    LscGeometry,
    LscKernel,
    ShBasisSpec,
    as_unit_directions,
    eval_basis,
    per_shell_operators,
)

_BACKENDS = (None, "auto", "numba", "numpy", "cuda")


def _dev(device=None):
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def _const(a, device) -> torch.Tensor:
    return torch.tensor(np.ascontiguousarray(a, dtype=np.float64), dtype=torch.float32, device=device).contiguous()


@dataclass(frozen=True)
class ShVolume:
    """(subjects, shells*R, X, Y, Z) SH coefficients on the device (fitting.py:33-60)."""

    data: torch.Tensor
    basis_spec: ShBasisSpec
    shells: int = 1

    def __post_init__(self) -> None:
        if self.data.dim() != 5:
            raise ShapeError(f"SH volume must be 5-D, got shape {tuple(self.data.shape)}")
        expected = self.shells * self.basis_spec.coeff_count
        if self.data.shape[1] != expected:
            raise ShapeError(f"SH volume has {self.data.shape[1]} channels, expected shells ({self.shells}) * R "
                             f"({self.basis_spec.coeff_count}) = {expected}")
        object.__setattr__(self, "data", ops.as_device_f32(self.data, "SH volume"))

    @property
    def grid_shape(self):
        return tuple(self.data.shape[2:])

    def shell_coeffs(self, shell: int) -> torch.Tensor:
        r = self.basis_spec.coeff_count
        return self.data[:, shell * r:(shell + 1) * r]


@dataclass(frozen=True)
class DwiVolume:
    """(subjects, shells*N, X, Y, Z) normalised signal on the device (fitting.py:63-89).

    check_finite=True repeats the reference's full-volume finiteness scan
    (fitting.py:80-81); it costs one extra pass over the volume and a host sync.
    """

    data: torch.Tensor
    shells: int = 1
    scheme: object = None          # dwio.GradientScheme of the channels, when known (fitting.py:69)
    check_finite: bool = True

    def __post_init__(self) -> None:
        if self.data.dim() != 5:
            raise ShapeError(f"DWI volume must be 5-D, got shape {tuple(self.data.shape)}")
        if self.shells < 1 or self.data.shape[1] % self.shells:
            raise ShapeError(f"channel count {self.data.shape[1]} is not divisible by shells = {self.shells}")
        t = ops.as_device_f32(self.data, "DWI volume")
        if self.check_finite and t.numel() and not bool(torch.isfinite(t).all()):
            raise ShapeError("DWI volume contains non-finite values")
        object.__setattr__(self, "data", t)

    @property
    def samples_per_shell(self) -> int:
        return self.data.shape[1] // self.shells

    @property
    def grid_shape(self):
        return tuple(self.data.shape[2:])


def _check_backend(backend) -> None:
    if backend not in _BACKENDS:
        raise ValueError(f"backend must be numba or numpy, got {backend!r}")


def signal_to_sh(vol: DwiVolume, op: FitOperator | Sequence[FitOperator], threads: int = 1) -> ShVolume:
    """Fit SH coefficients in every voxel; shared or per-shell operators (fitting.py:206-236)."""
    ops_ = per_shell_operators(op, vol.shells)
    n = ops_[0].n_gradients
    if vol.data.shape[1] != vol.shells * n:
        raise ShapeError(f"DWI volume has {vol.data.shape[1]} channels, expected shells ({vol.shells}) * N ({n}) = "
                         f"{vol.shells * n}")
    shared = all(o is ops_[0] for o in ops_)
    M = _const(np.stack([o.fit_matrix for o in (ops_[:1] if shared else ops_)]), vol.data.device)
    r = ops_[0].basis_spec.coeff_count
    out = ops.contract(vol.data, M, n, r, vol.shells, not shared)
    return ShVolume(out, ops_[0].basis_spec, vol.shells)


def sh_to_signal(sh: ShVolume, gradients, threads: int = 1) -> DwiVolume:
    """Evaluate every shell at arbitrary unit directions (fitting.py:239-250)."""
    dirs = as_unit_directions(gradients)
    B = _const(eval_basis(dirs, sh.basis_spec.order), sh.data.device)
    out = ops.contract(sh.data, B, sh.basis_spec.coeff_count, dirs.shape[0], sh.shells, False)
    return DwiVolume(out, sh.shells, check_finite=False)


def lsc_forward(sh_in: ShVolume, kernel: LscKernel, geom: LscGeometry, threads: int = 1,
                backend: str | None = None) -> ShVolume:
    """Local spherical convolution of an SH volume (lsc.py:158-199); same validation order."""
    _check_backend(backend)
    if sh_in.basis_spec.order != geom.order_in:
        raise ShapeError(f"SH input order {sh_in.basis_spec.order} does not match geometry input order "
                         f"{geom.order_in}")
    if kernel.shells_in != sh_in.shells:
        raise ShapeError(f"kernel expects {kernel.shells_in} input shells, volume has {sh_in.shells}")
    if kernel.kernel_len != geom.kernel_len:
        raise KernelMismatchError(f"kernel length K = {kernel.kernel_len} does not match geometry K = "
                                  f"{geom.kernel_len}")
    dev = sh_in.data.device
    fold, beta = _const(geom.fold, dev), _const(geom.beta, dev)
    w, b = _const(kernel.weights, dev), _const(kernel.bias, dev)
    L, _, bvec = ops.build_lsc_operator(fold, beta, w, b, want_Lt=False)
    r_in, r_out = geom.resample_matrix.shape[1], geom.refit.fit_matrix.shape[0]
    out = ops.contract(sh_in.data, L, kernel.shells_in * r_in, kernel.shells_out * r_out, 1, False, bias=bvec)
    return ShVolume(out, ShBasisSpec(geom.order_out), kernel.shells_out)


def apply_channel_matrix(matrix, stacked: torch.Tensor, threads: int = 1, out: torch.Tensor | None = None):
    """out[b, s] = matrix @ stacked[b, s] over (B, S, C_in, V) (fitting.py:155-188)."""
    if stacked.dim() != 4:
        raise ShapeError(f"stacked must be (B, S, C_in, V), got {tuple(stacked.shape)}")
    x = ops.as_device_f32(stacked, "stacked")
    W = matrix if isinstance(matrix, torch.Tensor) else _const(matrix, x.device)
    W = ops.as_device_f32(W, "matrix")
    c_out, c_in = W.shape
    nb, ns, ci, nv = x.shape
    if ci != c_in:
        raise ShapeError(f"matrix has {c_in} columns, stacked has {ci} channels")
    if out is not None and (tuple(out.shape) != (nb, ns, c_out, nv) or out.dtype != torch.float32
                            or not out.is_contiguous()):
        raise ShapeError("out must be a contiguous fp32 (B, S, C_out, V) tensor")
    y = ops.contract(x.view(nb, ns * c_in, nv), W, c_in, c_out, ns, False,
                     out=None if out is None else out.view(nb, ns * c_out, nv))
    return y.view(nb, ns, c_out, nv)


def lsc_combine(resample, weights, bias, coeffs: torch.Tensor, backend: str | None = None) -> torch.Tensor:
    """Origin values u[o,i,v] = bias[o] + sum_{s,k} w[o,s,k] (resample[iK+k] . coeffs[s,:,v]).

    The reference's kernel seam (_kernels.py:187-206).  Built as one contraction
    with Q_{o,s} = sum_k w[o,s,k] resample[k::K] -- the build_operator kernel
    with resample in place of the folded P_k and beta = 1.
    """
    _check_backend(backend)
    c = ops.as_device_f32(coeffs, "coeffs")
    if c.dim() != 3:
        raise ShapeError(f"coeffs must be (S_in, R_in, V), got {tuple(c.shape)}")
    w = np.asarray(weights, dtype=np.float64)
    s_out, s_in, K = w.shape
    rs = np.asarray(resample, dtype=np.float64)
    m = rs.shape[0] // K
    if rs.shape[0] != m * K or c.shape[0] != s_in or c.shape[1] != rs.shape[1]:
        raise ShapeError("lsc_combine: inconsistent shapes")
    dev = c.device
    P = _const(rs.reshape(m, K, -1).transpose(1, 0, 2), dev)        # (K, m, R_in)
    Q, _, bvec = ops.build_lsc_operator(P, _const(np.ones(m), dev), _const(w, dev),
                                        _const(np.asarray(bias, np.float64), dev), want_Lt=False)
    out = ops.contract(c.reshape(1, s_in * rs.shape[1], -1), Q, s_in * rs.shape[1], s_out * m, 1, False, bias=bvec)
    return out.view(s_out, m, -1)
