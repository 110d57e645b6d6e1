"""Device ops over the C ABI, with autograd.

Every op takes fp32 CUDA tensors in the reference's 5-D layout
(subjects, shells*C, X, Y, Z) and enqueues sm_100a kernels on the current
torch stream.  Non-CUDA input raises DeviceError: there is no CPU path.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import DeviceError, ShapeError

_NULL = ctypes.c_void_p(0)


def _stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t) -> ctypes.c_void_p:
    return _NULL if t is None else ctypes.c_void_p(t.data_ptr())


def as_device_f32(t: torch.Tensor, name: str) -> torch.Tensor:
    """fp32, contiguous, CUDA -- or DeviceError (no CPU fallback)."""
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor, got {type(t).__name__}")
    if not t.is_cuda:
        raise DeviceError(f"{name} must be a CUDA tensor on an sm_100a device; this implementation has no CPU path")
    if t.dtype != torch.float32:
        t = t.float()
    return t.contiguous()


def nvox_of(x: torch.Tensor) -> int:
    n = 1
    for d in x.shape[2:]:
        n *= int(d)
    return n


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


# ----------------------------------------------------------------------------- raw launchers
def contract(x: torch.Tensor, W: torch.Tensor, c_in: int, c_out: int, groups: int, per_group: bool,
             bias: torch.Tensor | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """out[b, g*c_out+i, v] = bias_g[i] + sum_j W_g[i,j] x[b, g*c_in+j, v]  (dl_chan_contract_f32)."""
    B = x.shape[0]
    if x.shape[1] != groups * c_in:
        raise ShapeError(f"expected {groups * c_in} channels, got {x.shape[1]}")
    if not (x.is_contiguous() and W.is_contiguous() and (bias is None or bias.is_contiguous())):
        raise ShapeError("contract: operands must be contiguous")
    if W.numel() != (groups if per_group else 1) * c_out * c_in:
        raise ShapeError(f"operator has {W.numel()} entries, expected {(groups if per_group else 1) * c_out * c_in}")
    V = nvox_of(x)
    if out is None:
        out = torch.empty((B, groups * c_out, *x.shape[2:]), dtype=torch.float32, device=x.device)
    _lib.call("dl_chan_contract_f32", _p(x), _p(out), _p(W), _p(bias), B, groups, c_in, c_out, V,
              groups * c_in * V, groups * c_out * V, int(per_group), _stream())
    return out


def build_lsc_operator(fold: torch.Tensor, beta: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None,
                       want_L=True, want_Lt=True, want_bvec=True):
    """(L, Lt, bvec) from the kernel parameters (dl_lsc_build_operator_f32)."""
    K, r_out, r_in = fold.shape
    s_out, s_in = weight.shape[0], weight.shape[1]
    dev = weight.device
    rows, cols = s_out * r_out, s_in * r_in
    L = torch.empty((rows, cols), dtype=torch.float32, device=dev) if want_L else None
    Lt = torch.empty((cols, rows), dtype=torch.float32, device=dev) if want_Lt else None
    bvec = torch.empty((rows,), dtype=torch.float32, device=dev) if want_bvec else None
    _lib.call("dl_lsc_build_operator_f32", _p(fold), _p(beta), _p(weight), _p(bias), _p(L), _p(Lt), _p(bvec),
              s_out, s_in, K, r_out, r_in, _stream())
    return L, Lt, bvec


def lsc_wgrad(g: torch.Tensor, c: torch.Tensor, fold: torch.Tensor, beta: torch.Tensor, s_out: int, s_in: int,
              want_dW=True, want_db=True):
    """(dW (s_out, s_in, K), db (s_out,)) = LSC parameter gradient (dl_lsc_wgrad_f32)."""
    K, r_out, r_in = fold.shape
    B, V = c.shape[0], nvox_of(c)
    dev = c.device
    dW = torch.empty((s_out, s_in, K), dtype=torch.float32, device=dev) if want_dW else None
    db = torch.empty((s_out,), dtype=torch.float32, device=dev) if want_db else None
    ws = _workspace(_lib.load().dl_lsc_wgrad_workspace_bytes(s_out, s_in, r_out, r_in), dev)
    _lib.call("dl_lsc_wgrad_f32", _p(g), _p(c), _p(fold), _p(beta), _p(dW), _p(db), _p(ws), B, s_out, s_in, K,
              r_out, r_in, V, s_out * r_out * V, s_in * r_in * V, _stream())
    return dW, db


def gemm_f64(A: torch.Tensor, B: torch.Tensor, ta: bool = False, tb: bool = False, C: torch.Tensor | None = None,
             alpha: float = 1.0, beta: float = 0.0) -> torch.Tensor:
    """C = alpha op(A) op(B) + beta C for small float64 device matrices (dl_gemm_f64, csrc/dense.cu)."""
    A, B = A.contiguous(), B.contiguous()
    m, k = (A.shape[1], A.shape[0]) if ta else (A.shape[0], A.shape[1])
    kb, n = (B.shape[1], B.shape[0]) if tb else (B.shape[0], B.shape[1])
    if kb != k:
        raise ShapeError(f"gemm_f64: inner dimensions {k} and {kb} differ")
    if C is None:
        C = torch.empty((m, n), dtype=torch.float64, device=A.device)
        beta = 0.0
    elif tuple(C.shape) != (m, n) or not C.is_contiguous():
        raise ShapeError("gemm_f64: C must be a contiguous (m, n) matrix")
    _lib.call("dl_gemm_f64", m, n, k, _p(A), A.shape[1], int(ta), _p(B), B.shape[1], int(tb), _p(C), n,
              ctypes.c_double(alpha), ctypes.c_double(beta), _stream())
    return C


def _affine(L: torch.Tensor, d: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """L d + b for float64 device vectors (one dl_gemm_f64 launch)."""
    return gemm_f64(L, d.reshape(-1, 1), C=b.clone().reshape(-1, 1), beta=1.0).reshape(-1)


# ----------------------------------------------------------------------------- autograd
class ChannelMap(torch.autograd.Function):
    """Per-shell linear map x[s] -> W_s x[s] (Signal2SH: W=M, SH2Signal: W=B'); grad uses W^T."""

    @staticmethod
    def forward(ctx, x, W, Wt, c_in, c_out, groups, per_group):
        ctx.save_for_backward(Wt)
        ctx.dims = (c_in, c_out, groups, per_group)
        return contract(x, W, c_in, c_out, groups, per_group)

    @staticmethod
    def backward(ctx, gy):
        (Wt,) = ctx.saved_tensors
        c_in, c_out, groups, per_group = ctx.dims
        gx = None
        if ctx.needs_input_grad[0]:
            gx = contract(as_device_f32(gy, "grad"), Wt, c_out, c_in, groups, per_group)
        return gx, None, None, None, None, None, None


class LscFunction(torch.autograd.Function):
    """Folded LSC: c_out = L(w) c_in + bias*beta; grads dc = L^T g, dW = <P_k, G>, db = beta.sum g."""

    @staticmethod
    def forward(ctx, c, weight, bias, fold, beta):
        s_out, s_in = weight.shape[0], weight.shape[1]
        K, r_out, r_in = fold.shape
        L, _, bvec = build_lsc_operator(fold, beta, weight, bias, want_Lt=False)
        out = contract(c, L, s_in * r_in, s_out * r_out, 1, False, bias=bvec)
        ctx.save_for_backward(c, weight, fold, beta)
        ctx.has_bias = bias is not None
        return out

    @staticmethod
    def backward(ctx, g):
        c, weight, fold, beta = ctx.saved_tensors
        s_out, s_in = weight.shape[0], weight.shape[1]
        K, r_out, r_in = fold.shape
        g = as_device_f32(g, "grad")
        dc = dW = db = None
        if ctx.needs_input_grad[0]:
            _, Lt, _ = build_lsc_operator(fold, beta, weight, None, want_L=False, want_bvec=False)
            dc = contract(g, Lt, s_out * r_out, s_in * r_in, 1, False)
        want_w = ctx.needs_input_grad[1]
        want_b = ctx.has_bias and ctx.needs_input_grad[2]
        if want_w or want_b:
            dW, db = lsc_wgrad(g, c, fold, beta, s_out, s_in, want_w, want_b)
            if dW is not None:
                dW = dW.view(weight.shape)
        return dc, dW, db, None, None


class ChainFunction(torch.autograd.Function):
    """Fused Signal2SH -> LSC -> SH2Signal on tcgen05 (dl_chain_fwd_f32 / dl_chain_bwd_f32).

    Forward is one kernel (x -> y) that also writes the Signal2SH coefficients c = M x as
    two-term bf16 planes (`c_mid`, the Gram operand) for the weight gradient; x itself is not
    kept.  Backward is one kernel for dx (the adjoint chain, which writes g = B'^T dy the same
    way to `g_mid`), one streaming Gram kernel over (g_mid, c_mid) for the LSC parameters, and
    a float64 finalize.
    """

    @staticmethod
    def forward(ctx, x, weight, bias, M, per_shell, fold, beta, Bt, state_fwd=None, state_bwd=None):
        s_out, s_in = weight.shape[0], weight.shape[1]
        K, r_out, r_in = fold.shape
        n = M.shape[-1]
        n_out = Bt.shape[0]
        B, V = x.shape[0], nvox_of(x)
        lib = _lib.load()
        want_w = ctx.needs_input_grad[1] or (bias is not None and ctx.needs_input_grad[2])
        L, _, bvec = build_lsc_operator(fold, beta, weight, bias, want_Lt=False)
        y = torch.empty((B, s_out * n_out, *x.shape[2:]), dtype=torch.float32, device=x.device)
        c_mid = _workspace(lib.dl_chain_mid_bytes(B, s_in, r_in, V), x.device) if want_w else None
        ws = _workspace(lib.dl_chain_workspace_bytes(B, s_in, s_out, n, r_in, r_out, n_out, V), x.device)
        _lib.call("dl_chain_fwd_f32", _p(x), _p(y), _p(c_mid), _p(M), int(per_shell), _p(L), _p(bvec), _p(Bt),
                  _p(ws), _p(state_fwd), B, s_in, s_out, n, r_in, r_out, n_out, V, _stream())
        ctx.save_for_backward(c_mid, weight, M, fold, beta, Bt, L)
        ctx.state_bwd = state_bwd
        ctx.per_shell = per_shell
        ctx.has_bias = bias is not None
        ctx.shape = (B, V, tuple(x.shape))
        return y

    @staticmethod
    def backward(ctx, dy):
        c_mid, weight, M, fold, beta, Bt, L = ctx.saved_tensors
        s_out, s_in = weight.shape[0], weight.shape[1]
        K, r_out, r_in = fold.shape
        n = M.shape[-1]
        n_out = Bt.shape[0]
        B, V, xshape = ctx.shape
        dy = as_device_f32(dy, "grad")
        want_x = ctx.needs_input_grad[0]
        want_w = ctx.needs_input_grad[1] and c_mid is not None
        want_b = ctx.has_bias and ctx.needs_input_grad[2] and c_mid is not None
        if not (want_x or want_w or want_b):
            return (None,) * 10
        lib = _lib.load()
        # the adjoint kernel always runs (it produces g for the Gram); without an input gradient it is told
        # dx = NULL and skips the dx stores (a g-only pass)
        dx = torch.empty(xshape, dtype=torch.float32, device=dy.device) if want_x else None
        dW = torch.empty((s_out, s_in, K), dtype=torch.float32, device=dy.device) if want_w else None
        db = torch.empty((s_out,), dtype=torch.float32, device=dy.device) if want_b else None
        g_mid = _workspace(lib.dl_chain_mid_bytes(B, s_out, r_out, V), dy.device) if (want_w or want_b) else None
        ws = _workspace(lib.dl_chain_workspace_bytes(B, s_in, s_out, n, r_in, r_out, n_out, V), dy.device)
        _lib.call("dl_chain_bwd_f32", _p(c_mid), _p(dy), _p(dx), _p(dW), _p(db), _p(g_mid), _p(M),
                  int(ctx.per_shell), _p(L), _p(Bt), _p(fold), _p(beta), _p(ws), _p(ctx.state_bwd), B, s_in, s_out, K,
                  n, r_in, r_out, n_out, V, _stream())
        if dW is not None:
            dW = dW.view(weight.shape)
        return (dx if want_x else None), dW, db, None, None, None, None, None, None, None


class RoundTripFunction(torch.autograd.Function):
    """Fused Signal2SH -> SH2Signal (dl_round_trip_fwd_f32 / dl_round_trip_bwd_f32).

    y[s] = B' M_s x[s] (fitting.py:206-250 composed): the coefficients c = M x stay in TMEM and the stage-2 product
    is block-diagonal over shells; the backward is the adjoint pass dx = M_s^T B'^T dy.
    """

    @staticmethod
    def forward(ctx, x, M, per_shell, Bt, shells, state_fwd, state_bwd):
        r, n = M.shape[-2], M.shape[-1]
        n_out = Bt.shape[0]
        B, V = x.shape[0], nvox_of(x)
        lib = _lib.load()
        y = torch.empty((B, shells * n_out, *x.shape[2:]), dtype=torch.float32, device=x.device)
        ws = _workspace(lib.dl_round_trip_workspace_bytes(B, shells, n, r, n_out, V), x.device)
        _lib.call("dl_round_trip_fwd_f32", _p(x), _p(y), _p(M), int(per_shell), _p(Bt), _p(ws), _p(state_fwd), B,
                  shells, n, r, n_out, V, _stream())
        ctx.save_for_backward(M, Bt)
        ctx.per_shell, ctx.state_bwd = per_shell, state_bwd
        ctx.shape = (B, V, tuple(x.shape), shells)
        return y

    @staticmethod
    def backward(ctx, dy):
        M, Bt = ctx.saved_tensors
        B, V, xshape, s = ctx.shape
        if not ctx.needs_input_grad[0]:
            return (None,) * 7
        r, n = M.shape[-2], M.shape[-1]
        n_out = Bt.shape[0]
        dy = as_device_f32(dy, "grad")
        lib = _lib.load()
        dx = torch.empty(xshape, dtype=torch.float32, device=dy.device)
        ws = _workspace(lib.dl_round_trip_workspace_bytes(B, s, n, r, n_out, V), dy.device)
        _lib.call("dl_round_trip_bwd_f32", _p(dy), _p(dx), _p(M), int(ctx.per_shell), _p(Bt), _p(ws), _p(ctx.state_bwd),
                  B, s, n, r, n_out, V, _stream())
        return dx, None, None, None, None, None, None


def chain_state(device) -> torch.Tensor:
    """Zeroed delayed-scaling state for one chain direction (dl_chain_state_bytes; kept across calls)."""
    return torch.zeros(int(_lib.load().dl_chain_state_bytes()) // 4, dtype=torch.int32, device=device)


class ChainStackFunction(torch.autograd.Function):
    """Fused Signal2SH -> LSC_1 -> ... -> LSC_n -> SH2Signal (n >= 2).

    The LSC layers are linear, so their product L = L_n ... L_1 and folded bias d_n (d_k = L_k d_{k-1} + bvec_k)
    run through the same fused kernels as one layer.  The backward asks the library for the float64 Gram
    G = sum_v g c^T and s = sum_v g (dl_chain_bwd_gram_f64); with A_k = L_{k+1}^T ... L_n^T and
    C_{k-1} = L_{k-1} ... L_1, layer k's operator gradient is A_k G C_{k-1}^T + (A_k s) d_{k-1}^T, giving
    dW_k = <P_k, .> and db_k = beta_k . A_k s -- no extra pass over the volume per layer.
    layers: (weight (S_out,S_in,K), bias or None, fold (K,R_out,R_in), beta (R_out,)) per layer, in order.
    """

    @staticmethod
    def forward(ctx, x, M, per_shell, Bt, state_fwd, state_bwd, n_layers, *layers):
        lib = _lib.load()
        ws_ = [layers[4 * i:4 * i + 4] for i in range(n_layers)]
        Ls, bvecs, L_tot, b_tot = _fold_layers(ws_)
        w1, f1 = ws_[0][0], ws_[0][2]
        wn, fn = ws_[-1][0], ws_[-1][2]
        s_in, r_in, s_out, r_out = w1.shape[1], f1.shape[2], wn.shape[0], fn.shape[1]
        n, n_out = M.shape[-1], Bt.shape[0]
        B, V = x.shape[0], nvox_of(x)
        want_w = any(ctx.needs_input_grad[7:])
        y = torch.empty((B, s_out * n_out, *x.shape[2:]), dtype=torch.float32, device=x.device)
        c_mid = _workspace(lib.dl_chain_mid_bytes(B, s_in, r_in, V), x.device) if want_w else None
        ws = _workspace(lib.dl_chain_workspace_bytes(B, s_in, s_out, n, r_in, r_out, n_out, V), x.device)
        _lib.call("dl_chain_fwd_f32", _p(x), _p(y), _p(c_mid), _p(M), int(per_shell), _p(L_tot), _p(b_tot), _p(Bt),
                  _p(ws), _p(state_fwd), B, s_in, s_out, n, r_in, r_out, n_out, V, _stream())
        ctx.save_for_backward(c_mid, M, Bt, L_tot, *[t for lay in ws_ for t in (lay[0], lay[2], lay[3])])
        ctx.Ls, ctx.bvecs = Ls, bvecs
        ctx.dims = (s_in, s_out, n, r_in, r_out, n_out, B, V, tuple(x.shape), n_layers)
        ctx.has_bias = [lay[1] is not None for lay in ws_]
        ctx.per_shell, ctx.state_bwd = per_shell, state_bwd
        return y

    @staticmethod
    def backward(ctx, dy):
        c_mid, M, Bt, L_tot, *lay = ctx.saved_tensors
        s_in, s_out, n, r_in, r_out, n_out, B, V, xshape, nl = ctx.dims
        lib = _lib.load()
        dy = as_device_f32(dy, "grad")
        nones = [None] * (7 + 4 * nl)
        if c_mid is None and not ctx.needs_input_grad[0]:
            return tuple(nones)
        dx = torch.empty(xshape, dtype=torch.float32, device=dy.device) if ctx.needs_input_grad[0] else None
        ws = _workspace(lib.dl_chain_workspace_bytes(B, s_in, s_out, n, r_in, r_out, n_out, V), dy.device)
        rows, cols = ctypes.c_int64(), ctypes.c_int64()
        _lib.call("dl_chain_gram_dims", s_in, s_out, r_in, r_out, ctypes.byref(rows), ctypes.byref(cols))
        if c_mid is None:   # dx only: the single-layer entry with no weight gradient
            _lib.call("dl_chain_bwd_f32", _NULL, _p(dy), _p(dx), _NULL, _NULL, _NULL, _p(M), int(ctx.per_shell),
                      _p(L_tot), _p(Bt), _NULL, _NULL, _p(ws), _p(ctx.state_bwd), B, s_in, s_out, 1, n, r_in, r_out,
                      n_out, V, _stream())
            out = list(nones)
            out[0] = dx
            return tuple(out)
        G = torch.empty((rows.value, cols.value), dtype=torch.float64, device=dy.device)
        g_mid = _workspace(lib.dl_chain_mid_bytes(B, s_out, r_out, V), dy.device)
        _lib.call("dl_chain_bwd_gram_f64", _p(c_mid), _p(dy), _p(dx), _p(G), _p(g_mid), _p(M), int(ctx.per_shell),
                  _p(L_tot), _p(Bt), _p(ws), _p(ctx.state_bwd), B, s_in, s_out, n, r_in, r_out, n_out, V, _stream())
        grads = _layer_grads(G, rows.value, cols.value, (s_in, s_out, r_in, r_out, nl), ctx.Ls, ctx.bvecs, lay,
                             ctx.has_bias, dy.device)
        out = list(nones)
        out[0] = dx if ctx.needs_input_grad[0] else None
        for k in range(nl):
            out[7 + 4 * k] = grads[2 * k]
            out[7 + 4 * k + 1] = grads[2 * k + 1]
        return tuple(out)


def _fold_layers(layers):
    """Per-layer (L_k, bvec_k) in float64 and the product L = L_n ... L_1 with its folded bias (dl_gemm_f64)."""
    Ls, bvecs = [], []
    for w, b, fold, beta in layers:
        L, _, bvec = build_lsc_operator(fold, beta, w, b, want_Lt=False)
        Ls.append(L.double())
        bvecs.append(bvec.double())
    Lt, dt = Ls[0], bvecs[0]
    for L, bv in zip(Ls[1:], bvecs[1:]):
        Lt, dt = gemm_f64(L, Lt), _affine(L, dt, bv)
    return Ls, bvecs, Lt.float().contiguous(), dt.float().contiguous()


def _layer_grads(G, rows, cols, dims, Ls, bvecs, lay, has_bias, device):
    """Per-layer dW / db from the float64 Gram (see ChainStackFunction); `lay` = (w, fold, beta) per layer.
    dL_k = A_k G C_{k-1}^T + (A_k s) d_{k-1}^T by dl_gemm_f64, dW_k = <P_k, dL_k> by dl_lsc_dw_from_dl_f64."""
    s_in, s_out, r_in, r_out, nl = dims
    rpo, rpi = rows // s_out, cols // s_in
    Gr = G.view(s_out, rpo, s_in, rpi)[:, :r_out, :, :r_in].reshape(s_out * r_out, s_in * r_in).contiguous()
    sv = G.view(s_out, rpo, cols)[:, :r_out, r_in].reshape(-1).contiguous()
    Cs, ds = [None] * nl, [None] * nl
    C = torch.eye(s_in * r_in, dtype=torch.float64, device=device)
    d = torch.zeros(s_in * r_in, dtype=torch.float64, device=device)
    for k in range(nl):
        Cs[k], ds[k] = C, d
        if k + 1 < nl:
            C, d = gemm_f64(Ls[k], C), _affine(Ls[k], d, bvecs[k])
    out = [None] * (2 * nl)
    A = torch.eye(s_out * r_out, dtype=torch.float64, device=device)
    for k in reversed(range(nl)):
        w, fold, beta = lay[3 * k], lay[3 * k + 1], lay[3 * k + 2]
        so, si, K = w.shape
        ro, ri = fold.shape[1], fold.shape[2]
        gs = gemm_f64(A, sv.reshape(-1, 1)).reshape(-1)
        dL = gemm_f64(gemm_f64(A, Gr), Cs[k], tb=True)
        dL = gemm_f64(gs.reshape(-1, 1), ds[k].reshape(1, -1), C=dL, beta=1.0)
        dW = torch.empty((so, si, K), dtype=torch.float32, device=device)
        _lib.call("dl_lsc_dw_from_dl_f64", _p(dL), _p(fold), _p(dW), so, si, K, ro, ri, _stream())
        out[2 * k] = dW
        if has_bias[k]:
            out[2 * k + 1] = gemm_f64(gs.reshape(so, ro), beta.double().reshape(-1, 1)).reshape(-1).float()
        if k > 0:
            A = gemm_f64(Ls[k], A, ta=True)
    return out


class ChainMseFunction(torch.autograd.Function):
    """mean((chain(x) - target)^2) with the loss and its gradient fused into the forward kernel.

    dl_chain_fwd_mse_f32 writes dy = 2 (y - target) / numel(y) in place of y and reduces the loss; the
    backward runs the adjoint on that dy (g-only when x needs no gradient) and takes every layer's dW / db from
    the one float64 Gram.  One or more LSC layers (folded as in ChainStackFunction).
    """

    @staticmethod
    def forward(ctx, x, target, M, per_shell, Bt, state_fwd, state_bwd, n_layers, *layers):
        lib = _lib.load()
        lays = [layers[4 * i:4 * i + 4] for i in range(n_layers)]
        Ls, bvecs, L_tot, b_tot = _fold_layers(lays)
        w1, f1, wn, fn = lays[0][0], lays[0][2], lays[-1][0], lays[-1][2]
        s_in, r_in, s_out, r_out = w1.shape[1], f1.shape[2], wn.shape[0], fn.shape[1]
        n, n_out = M.shape[-1], Bt.shape[0]
        B, V = x.shape[0], nvox_of(x)
        if tuple(target.shape) != (B, s_out * n_out, *x.shape[2:]):
            raise ShapeError(f"target has shape {tuple(target.shape)}, the chain output is "
                             f"{(B, s_out * n_out, *x.shape[2:])}")
        target = as_device_f32(target, "target")
        want_w = any(ctx.needs_input_grad[8:])
        dy = torch.empty((B, s_out * n_out, *x.shape[2:]), dtype=torch.float32, device=x.device)
        loss = torch.zeros(4, dtype=torch.float64, device=x.device)
        c_mid = _workspace(lib.dl_chain_mid_bytes(B, s_in, r_in, V), x.device) if want_w else None
        ws = _workspace(lib.dl_chain_workspace_bytes(B, s_in, s_out, n, r_in, r_out, n_out, V), x.device)
        _lib.call("dl_chain_fwd_mse_f32", _p(x), _p(target), _p(dy), _p(c_mid), _p(M), int(per_shell), _p(L_tot),
                  _p(b_tot), _p(Bt), _p(ws), _p(state_fwd), _p(loss), B, s_in, s_out, n, r_in, r_out, n_out, V,
                  _stream())
        ctx.save_for_backward(c_mid, dy, M, Bt, L_tot, *[t for lay in lays for t in (lay[0], lay[2], lay[3])])
        ctx.Ls, ctx.bvecs = Ls, bvecs
        ctx.dims = (s_in, s_out, n, r_in, r_out, n_out, B, V, tuple(x.shape), n_layers)
        ctx.has_bias = [lay[1] is not None for lay in lays]
        ctx.per_shell, ctx.state_bwd = per_shell, state_bwd
        return loss[2].float()

    @staticmethod
    def backward(ctx, g):
        c_mid, dy, M, Bt, L_tot, *lay = ctx.saved_tensors
        s_in, s_out, n, r_in, r_out, n_out, B, V, xshape, nl = ctx.dims
        lib = _lib.load()
        out = [None] * (8 + 4 * nl)
        want_x = ctx.needs_input_grad[0]
        if ctx.needs_input_grad[1]:
            out[1] = -dy * g
        if c_mid is None and not want_x:
            return tuple(out)
        dx = torch.empty(xshape, dtype=torch.float32, device=dy.device) if want_x else None
        ws = _workspace(lib.dl_chain_workspace_bytes(B, s_in, s_out, n, r_in, r_out, n_out, V), dy.device)
        if c_mid is None:
            _lib.call("dl_chain_bwd_f32", _NULL, _p(dy), _p(dx), _NULL, _NULL, _NULL, _p(M), int(ctx.per_shell),
                      _p(L_tot), _p(Bt), _NULL, _NULL, _p(ws), _p(ctx.state_bwd), B, s_in, s_out, 1, n, r_in, r_out,
                      n_out, V, _stream())
        else:
            rows, cols = ctypes.c_int64(), ctypes.c_int64()
            _lib.call("dl_chain_gram_dims", s_in, s_out, r_in, r_out, ctypes.byref(rows), ctypes.byref(cols))
            G = torch.empty((rows.value, cols.value), dtype=torch.float64, device=dy.device)
            g_mid = _workspace(lib.dl_chain_mid_bytes(B, s_out, r_out, V), dy.device)
            _lib.call("dl_chain_bwd_gram_f64", _p(c_mid), _p(dy), _p(dx), _p(G), _p(g_mid), _p(M),
                      int(ctx.per_shell), _p(L_tot), _p(Bt), _p(ws), _p(ctx.state_bwd), B, s_in, s_out, n, r_in, r_out,
                      n_out, V, _stream())
            grads = _layer_grads(G, rows.value, cols.value, (s_in, s_out, r_in, r_out, nl), ctx.Ls, ctx.bvecs, lay,
                                 ctx.has_bias, dy.device)
            for k in range(nl):
                if ctx.needs_input_grad[8 + 4 * k] and grads[2 * k] is not None:
                    out[8 + 4 * k] = grads[2 * k] * g
                if ctx.needs_input_grad[8 + 4 * k + 1] and grads[2 * k + 1] is not None:
                    out[8 + 4 * k + 1] = grads[2 * k + 1] * g
        if want_x:
            out[0] = dx * g
        return tuple(out)


def chain_mse_supported(s_in: int, s_out: int, n: int, r_in: int, r_out: int, n_out: int, per_shell: bool) -> bool:
    """True if the fused-loss forward (dl_chain_fwd_mse_f32) covers these channel counts."""
    return bool(_lib.load().dl_chain_mse_supported(s_in, s_out, n, r_in, r_out, n_out, int(per_shell)))


def fp16_pass_enabled() -> bool:
    """True when the fused chain runs the fp16 two-term pass (the default precision mode)."""
    import os

    return "DELIMIT_SPLIT_TERMS" not in os.environ


def chain_supported(s_in: int, s_out: int, n: int, r_in: int, r_out: int, n_out: int, per_shell: bool) -> bool:
    """True if the fused tcgen05 chain kernels fit these channel counts."""
    return bool(_lib.load().dl_chain_supported(s_in, s_out, n, r_in, r_out, n_out, int(per_shell)))
