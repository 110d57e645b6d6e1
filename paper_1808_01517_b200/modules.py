"""DELIMIT layers as torch.nn.Modules (the paper's API).

* Signal2SH(sh_order, gradients, lb_lambda=0.0, shells=None)
* SH2Signal(sh_order, gradients)
* LocalSphericalConvolution(shells_in, shells_out, sh_order_in, sh_order_out, sampled_gradients,
                            kernel_sizes, lb_lambda=0.006, angular_distance=pi/5)
  with .sconv.weight (shells_out, shells_in, 1, K) and .sconv.bias (shells_out,)
* SphericalChain(s2sh, lsc, sh2s): the three fused into one forward and one backward pass.
* RoundTrip(s2sh, sh2s): Signal2SH -> SH2Signal fused (the coefficients never reach HBM).

Tensors are 5-D subjects x (shells*gradients) x H x W x D, fp32 CUDA.
Operators are built once per gradient table on the host in float64 (geometry.py)
and held as fp32 device buffers; the per-voxel work runs in the sm_100a kernels.
"""

from __future__ import annotations

import math

import numpy as np
import torch
from torch import nn

from . import ops
from .errors import KernelMismatchError, ShapeError
from .geometry import (
    LscKernel,
    build_lsc_geometry,
    coeff_count,
    eval_basis,
    make_fit_operator,
    seq_or_single,
)


def _f32(a) -> torch.Tensor:
    return torch.tensor(np.ascontiguousarray(a, dtype=np.float64), dtype=torch.float32).contiguous()


def _check_5d(x: torch.Tensor, what: str) -> None:
    if x.dim() != 5:
        raise ShapeError(f"{what} must be 5-D (subjects, shells*C, X, Y, Z), got shape {tuple(x.shape)}")


class Signal2SH(nn.Module):
    """Signal -> SH coefficients per shell: c[s] = M_s x[s] (fitting.signal_to_sh, fitting.py:206-236).

    gradients: (N, 3) shared by every shell, or (S, N, 3) one table per shell.
    shells: optional fixed shell count; by default inferred as channels / N.
    """

    def __init__(self, sh_order: int, gradients, lb_lambda: float = 0.0, shells: int | None = None):
        super().__init__()
        tables, per_shell = seq_or_single(gradients)
        self.operators = [make_fit_operator(t, sh_order, lb_lambda) for t in tables]
        if len({op.n_gradients for op in self.operators}) != 1:
            raise ShapeError("per-shell fit operators must share one gradient count")
        self.sh_order = int(sh_order)
        self.lb_lambda = float(lb_lambda)
        self.n_gradients = self.operators[0].n_gradients
        self.n_coeffs = coeff_count(sh_order)
        self.per_shell = per_shell
        self.shells = len(tables) if per_shell else shells
        M = np.stack([op.fit_matrix for op in self.operators])            # (S|1, R, N)
        self.register_buffer("fit_matrix", _f32(M), persistent=False)
        self.register_buffer("fit_matrix_t", _f32(np.transpose(M, (0, 2, 1))), persistent=False)

    def n_shells(self, channels: int) -> int:
        if channels % self.n_gradients:
            raise ShapeError(f"signal has {channels} channels, not a multiple of N = {self.n_gradients}")
        s = channels // self.n_gradients
        if self.shells is not None and s != self.shells:
            raise ShapeError(f"signal has {channels} channels, expected shells ({self.shells}) * N "
                             f"({self.n_gradients}) = {self.shells * self.n_gradients}")
        return s

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        _check_5d(x, "signal")
        s = self.n_shells(x.shape[1])
        x = ops.as_device_f32(x, "signal")
        return ops.ChannelMap.apply(x, self.fit_matrix, self.fit_matrix_t, self.n_gradients, self.n_coeffs, s,
                                    self.per_shell)

    def extra_repr(self) -> str:
        return f"sh_order={self.sh_order}, n_gradients={self.n_gradients}, lb_lambda={self.lb_lambda}"


class SH2Signal(nn.Module):
    """SH coefficients -> signal at `gradients` per shell: y[s] = B' c[s] (fitting.py:239-250).

    The basis is evaluated once here, not per call as the reference does (fitting.py:242).
    """

    def __init__(self, sh_order: int, gradients):
        super().__init__()
        B = eval_basis(gradients, sh_order)                                # (N, R)
        self.sh_order = int(sh_order)
        self.n_gradients, self.n_coeffs = B.shape
        self.register_buffer("basis", _f32(B), persistent=False)
        self.register_buffer("basis_t", _f32(B.T), persistent=False)

    def forward(self, c: torch.Tensor) -> torch.Tensor:
        _check_5d(c, "SH volume")
        if c.shape[1] % self.n_coeffs:
            raise ShapeError(f"SH volume has {c.shape[1]} channels, not a multiple of R = {self.n_coeffs}")
        s = c.shape[1] // self.n_coeffs
        c = ops.as_device_f32(c, "SH volume")
        return ops.ChannelMap.apply(c, self.basis, self.basis_t, self.n_coeffs, self.n_gradients, s, False)

    def extra_repr(self) -> str:
        return f"sh_order={self.sh_order}, n_gradients={self.n_gradients}"


class SphericalKernel(nn.Module):
    """Holds the LSC parameters with the paper's shapes: weight (S_out, S_in, 1, K), bias (S_out,)."""

    def __init__(self, shells_in: int, shells_out: int, kernel_len: int):
        super().__init__()
        self.weight = nn.Parameter(torch.empty(shells_out, shells_in, 1, kernel_len))
        self.bias = nn.Parameter(torch.empty(shells_out))
        bound = 1.0 / math.sqrt(shells_in * kernel_len)     # nn.Conv2d's default fan-in init
        with torch.no_grad():
            self.weight.uniform_(-bound, bound)
            self.bias.uniform_(-bound, bound)


class LocalSphericalConvolution(nn.Module):
    """Ring-kernel local spherical convolution (lsc.lsc_forward, lsc.py:158-199).

    Per voxel: resample each input shell on origin + rings, cross-correlate with
    the ring kernel, add the bias, refit at sh_order_out.  Executed as the
    equivalent folded operator L(w) = sum_k w[o,s,k] P_k (one kernel launch).
    """

    def __init__(self, shells_in: int, shells_out: int, sh_order_in: int, sh_order_out: int, sampled_gradients,
                 kernel_sizes, lb_lambda: float = 0.006, angular_distance: float = math.pi / 5):
        super().__init__()
        self.geometry = build_lsc_geometry(sampled_gradients, kernel_sizes, angular_distance, sh_order_in,
                                           sh_order_out, lb_lambda)
        self.shells_in, self.shells_out = int(shells_in), int(shells_out)
        self.sh_order_in, self.sh_order_out = int(sh_order_in), int(sh_order_out)
        self.kernel_sizes = tuple(self.geometry.kernel_sizes)
        self.angular_distance = float(angular_distance)
        self.lb_lambda = float(lb_lambda)
        self.kernel_len = self.geometry.kernel_len
        self.r_in, self.r_out = coeff_count(sh_order_in), coeff_count(sh_order_out)
        self.sconv = SphericalKernel(self.shells_in, self.shells_out, self.kernel_len)
        self.register_buffer("fold", _f32(self.geometry.fold), persistent=False)     # (K, R_out, R_in)
        self.register_buffer("beta", _f32(self.geometry.beta), persistent=False)     # (R_out,)

    # -- parameter interchange with the reference's LscKernel --------------------------------------
    @property
    def kernel(self) -> LscKernel:
        w = self.sconv.weight.detach().double().cpu().numpy()[:, :, 0, :]
        b = self.sconv.bias.detach().double().cpu().numpy()
        return LscKernel(weights=w, bias=b)

    def load_kernel(self, kernel: LscKernel) -> None:
        if kernel.kernel_len != self.kernel_len:
            raise KernelMismatchError(f"kernel length K = {kernel.kernel_len} does not match geometry K = "
                                      f"{self.kernel_len}")
        if (kernel.shells_out, kernel.shells_in) != (self.shells_out, self.shells_in):
            raise ShapeError(f"kernel is {kernel.shells_out}x{kernel.shells_in} shells, layer is "
                             f"{self.shells_out}x{self.shells_in}")
        with torch.no_grad():
            self.sconv.weight.copy_(torch.as_tensor(kernel.weights[:, :, None, :]))
            self.sconv.bias.copy_(torch.as_tensor(kernel.bias))

    def _validate(self, c: torch.Tensor) -> None:
        _check_5d(c, "SH volume")
        w = self.sconv.weight
        if w.dim() != 4 or w.shape[2] != 1:
            raise ShapeError(f"sconv.weight must be (shells_out, shells_in, 1, K), got {tuple(w.shape)}")
        if w.shape[3] != self.kernel_len:
            raise KernelMismatchError(f"kernel length K = {w.shape[3]} does not match geometry K = {self.kernel_len}")
        if c.shape[1] % self.r_in:
            raise ShapeError(f"SH input order does not match: {c.shape[1]} channels is not a multiple of "
                             f"R_in = {self.r_in} (order {self.sh_order_in})")
        if c.shape[1] // self.r_in != w.shape[1]:
            raise ShapeError(f"kernel expects {w.shape[1]} input shells, volume has {c.shape[1] // self.r_in}")
        if self.sconv.bias is not None and self.sconv.bias.shape != (w.shape[0],):
            raise ShapeError(f"bias must have one entry per output shell, got {tuple(self.sconv.bias.shape)}")

    def forward(self, c: torch.Tensor) -> torch.Tensor:
        self._validate(c)
        c = ops.as_device_f32(c, "SH volume")
        w = self.sconv.weight
        w3 = w.reshape(w.shape[0], w.shape[1], w.shape[3])
        if w3.dtype != torch.float32:
            w3 = w3.float()
        b = self.sconv.bias
        return ops.LscFunction.apply(c, w3.contiguous(), None if b is None else b.float().contiguous(),
                                     self.fold, self.beta)

    def extra_repr(self) -> str:
        return (f"shells_in={self.shells_in}, shells_out={self.shells_out}, sh_order_in={self.sh_order_in}, "
                f"sh_order_out={self.sh_order_out}, kernel_sizes={list(self.kernel_sizes)}, "
                f"angular_distance={self.angular_distance:.6g}, lb_lambda={self.lb_lambda}")


class SphericalChain(nn.Module):
    """Signal2SH -> LocalSphericalConvolution -> SH2Signal as ONE fused op (forward + backward).

    Equivalent to sh2s(lsc(s2sh(x))) -- the chain the reference CLI runs (cli.py:159-245) --
    with the LSC parameters shared with `lsc`.  The fused path runs the whole chain in one
    tcgen05 kernel per direction (intermediates stay in TMEM); channel counts beyond the
    kernels' TMEM/shared-memory plan run the three layers one after the other instead.
    """

    def __init__(self, s2sh: Signal2SH, lsc, sh2s: SH2Signal):
        super().__init__()
        layers = [lsc] if isinstance(lsc, LocalSphericalConvolution) else list(lsc)
        if not layers or not all(isinstance(m, LocalSphericalConvolution) for m in layers):
            raise ShapeError("lsc must be a LocalSphericalConvolution or a non-empty sequence of them")
        first, last = layers[0], layers[-1]
        if s2sh.sh_order != first.sh_order_in:
            raise ShapeError(f"Signal2SH order {s2sh.sh_order} does not match LSC input order {first.sh_order_in}")
        if sh2s.sh_order != last.sh_order_out:
            raise ShapeError(f"SH2Signal order {sh2s.sh_order} does not match LSC output order {last.sh_order_out}")
        if s2sh.per_shell and len(s2sh.operators) != first.shells_in:
            raise ShapeError(f"Signal2SH has {len(s2sh.operators)} shell operators, LSC expects {first.shells_in}")
        for a, b in zip(layers, layers[1:]):
            if (a.shells_out, a.sh_order_out) != (b.shells_in, b.sh_order_in):
                raise ShapeError(f"LSC layers do not chain: {a.shells_out} shells of order {a.sh_order_out} into "
                                 f"{b.shells_in} shells of order {b.sh_order_in}")
        # one layer: `lsc` is that module (as before); several: an nn.ModuleList in order
        self.s2sh, self.sh2s = s2sh, sh2s
        self.lsc = layers[0] if len(layers) == 1 else nn.ModuleList(layers)
        self._layers = layers
        self._fused = None
        self._state = {}   # device -> (forward, adjoint) delayed-scaling state of the fp16 chain pass

    def range_state(self, device):
        """The (forward, adjoint) scale-history tensors of the fused kernels on `device` (ops.chain_state).

        The kernels read and update this state in place, so one module instance must not run on two streams
        at once: concurrent calls would share the range record, and one call's in-range record could hide the
        other's out-of-range fp16 pass.  Use one instance per concurrent stream.  (The state is deliberately
        not keyed by stream: CUDA-graph capture runs on a side stream, and a state created inside the capture
        would be re-zeroed by every replay.)"""
        key = str(device)
        if key not in self._state:
            self._state[key] = (ops.chain_state(device), ops.chain_state(device))
        return self._state[key]

    def mse_loss(self, x: torch.Tensor, target: torch.Tensor, fused: bool = True) -> torch.Tensor:
        """mean((self(x) - target)^2).

        fused=True (default, when the channel counts allow) computes the loss and its gradient inside the
        forward kernel (ops.ChainMseFunction: dy is written in place of y, y is never stored); fused=False is
        the chain output and torch's MSE (the fused forward streams the target through per-warp rings).
        """
        first, last = self._layers[0], self._layers[-1]
        if not (fused and self.fused() and ops.chain_mse_supported(first.shells_in, last.shells_out,
                                                                   self.s2sh.n_gradients, first.r_in, last.r_out,
                                                                   self.sh2s.n_gradients, self.s2sh.per_shell)):
            return torch.nn.functional.mse_loss(self(x), target)
        _check_5d(x, "signal")
        s = self.s2sh.n_shells(x.shape[1])
        if s != first.shells_in:
            raise ShapeError(f"kernel expects {first.shells_in} input shells, volume has {s}")
        shells = s
        for layer in self._layers:
            layer._validate(torch.empty((1, shells * layer.r_in, 1, 1, 1), device="meta"))
            shells = layer.shells_out
        x = ops.as_device_f32(x, "signal")
        sf, sb = self.range_state(x.device)
        args = []
        for layer in self._layers:
            w, b = layer.sconv.weight, layer.sconv.bias
            args += [w.reshape(w.shape[0], w.shape[1], w.shape[3]).float().contiguous(),
                     None if b is None else b.float().contiguous(), layer.fold, layer.beta]
        return ops.ChainMseFunction.apply(x, target, self.s2sh.fit_matrix, self.s2sh.per_shell, self.sh2s.basis, sf,
                                          sb, len(self._layers), *args)

    def fused(self) -> bool:
        if self._fused is None:
            first, last = self._layers[0], self._layers[-1]
            self._fused = ops.chain_supported(first.shells_in, last.shells_out, self.s2sh.n_gradients,
                                              first.r_in, last.r_out, self.sh2s.n_gradients, self.s2sh.per_shell)
        return self._fused

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        _check_5d(x, "signal")
        first = self._layers[0]
        s = self.s2sh.n_shells(x.shape[1])
        if s != first.shells_in:
            raise ShapeError(f"kernel expects {first.shells_in} input shells, volume has {s}")
        shells = s
        for layer in self._layers:
            layer._validate(torch.empty((1, shells * layer.r_in, 1, 1, 1), device="meta"))
            shells = layer.shells_out
        x = ops.as_device_f32(x, "signal")
        if not self.fused():
            u = self.s2sh(x)
            for layer in self._layers:
                u = layer(u)
            return self.sh2s(u)
        if len(self._layers) > 1:
            sf, sb = self.range_state(x.device)
            args = []
            for layer in self._layers:
                w = layer.sconv.weight
                b = layer.sconv.bias
                args += [w.reshape(w.shape[0], w.shape[1], w.shape[3]).float().contiguous(),
                         None if b is None else b.float().contiguous(), layer.fold, layer.beta]
            return ops.ChainStackFunction.apply(x, self.s2sh.fit_matrix, self.s2sh.per_shell, self.sh2s.basis, sf,
                                                sb, len(self._layers), *args)
        w = self.lsc.sconv.weight
        w3 = w.reshape(w.shape[0], w.shape[1], w.shape[3]).float().contiguous()
        b = self.lsc.sconv.bias
        sf, sb = self.range_state(x.device)
        return ops.ChainFunction.apply(x, w3, None if b is None else b.float().contiguous(),
                                       self.s2sh.fit_matrix, self.s2sh.per_shell, self.lsc.fold, self.lsc.beta,
                                       self.sh2s.basis, sf, sb)


class RoundTrip(nn.Module):
    """Signal2SH -> SH2Signal as ONE fused op (forward + backward): y[s] = B' M_s x[s].

    Equivalent to sh2s(s2sh(x)) -- signal_to_sh then sh_to_signal (fitting.py:206-250), the round trip of the
    reference's acceptance criterion 1 -- run through the fused chain kernels with the identity in place of
    the LSC operator, so the SH coefficients stay in tensor memory.  Channel counts outside the fused plan run
    the two layers one after the other.
    """

    def __init__(self, s2sh: Signal2SH, sh2s: SH2Signal):
        super().__init__()
        if s2sh.sh_order != sh2s.sh_order:
            raise ShapeError(f"Signal2SH order {s2sh.sh_order} does not match SH2Signal order {sh2s.sh_order}")
        self.s2sh, self.sh2s = s2sh, sh2s
        self._state = {}
        self._fused = {}

    def range_state(self, device):
        """(forward, adjoint) delayed-scaling state of the fused kernels on `device` (single-stream use, as
        SphericalChain.range_state)."""
        key = str(device)
        if key not in self._state:
            self._state[key] = (ops.chain_state(device), ops.chain_state(device))
        return self._state[key]

    def fused(self, shells: int) -> bool:
        if shells not in self._fused:
            r = self.s2sh.n_coeffs
            self._fused[shells] = ops.chain_supported(shells, shells, self.s2sh.n_gradients, r, r,
                                                      self.sh2s.n_gradients, self.s2sh.per_shell)
        return self._fused[shells]

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        _check_5d(x, "signal")
        s = self.s2sh.n_shells(x.shape[1])
        x = ops.as_device_f32(x, "signal")
        if not self.fused(s):
            return self.sh2s(self.s2sh(x))
        sf, sb = self.range_state(x.device)
        return ops.RoundTripFunction.apply(x, self.s2sh.fit_matrix, self.s2sh.per_shell, self.sh2s.basis, s, sf, sb)
