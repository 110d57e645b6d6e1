"""Raw acquisition -> normalised 5-D signal on the device.

normalize_b0(raw, bvals_or_scheme, b0_threshold, tolerance, shells) keeps the reference's signature and
errors (fitting.py:253-342): mean b0 per voxel, exclusion below 1e-6 of its maximum, division, shell-blocked
channel order, (1, shells * m, X, Y, Z) output plus the (X, Y, Z) exclusion mask.  The arithmetic runs in
one fused kernel (dl_normalize_b0_f32, csrc/ingest.cu) that reads the acquisition in its stored layout and
type -- an (X, Y, Z, V) array of any dtype the NIfTI reader supports, or a NIfTI file's own bytes -- so
the b0 mean, scaling, division and the move to channel-major order cost one pass over HBM.

load_dwi(nifti, bvals, bvecs, ...) goes from files to the hot path's input: the voxel bytes are read once
(dwio.read_nifti_raw), staged in pinned memory, copied to the device as stored and normalised there.

chain_from_raw(chain, raw, bvals_or_scheme, ...) fuses the normalisation INTO the chain:
the fused Signal2SH -> LSC -> SH2Signal kernel reads the acquisition's stored volumes (int16 / float32, x fastest)
and applies x = raw * slope / mean_b0 in its input role (dl_chain_fwd_raw_f32), so the normalised volume never
exists; the output comes back in the acquisition's voxel order as a (1, C, X, Y, Z) view -- exactly the layout a
NIfTI file of the result stores.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np
import torch

from . import _lib, dwio
from .errors import MissingB0Error, ShapeError
from .functional import DwiVolume
from .ops import _p, _stream

_CODE_OF_TORCH = {torch.uint8: 2, torch.int16: 4, torch.int32: 8, torch.float32: 16, torch.float64: 64}
_TORCH_OF = {np.uint8: torch.uint8, np.int16: torch.int16, np.int32: torch.int32, np.float32: torch.float32,
             np.float64: torch.float64}


def select_volumes(bvals_or_scheme, nvol: int, b0_threshold: float = dwio.B0_THRESHOLD,
                   tolerance: float = dwio.SHELL_TOLERANCE, shells: Sequence[float] | None = None):
    """(b0 indices, chosen shells) with the reference's checks and messages (fitting.py:276-311)."""
    if isinstance(bvals_or_scheme, dwio.GradientScheme):
        b0_idx, table = bvals_or_scheme.b0_indices, bvals_or_scheme.shells
    else:
        b0_idx, table = dwio.detect_shells(np.asarray(bvals_or_scheme, dtype=np.float64), tolerance=tolerance,
                                           b0_threshold=b0_threshold)
    covered = b0_idx.size + sum(s.indices.size for s in table)
    if covered != nvol:
        raise ShapeError(f"gradient table describes {covered} volumes, data has {nvol}")
    if b0_idx.size == 0:
        raise MissingB0Error("acquisition has no b=0 volume to normalize against")
    if shells is not None:
        table = tuple(dwio.nearest_shell(table, want, tolerance) for want in shells)
    if not table:
        raise ShapeError("no diffusion-weighted shells selected")
    if len({s.indices.size for s in table}) != 1:
        raise ShapeError("shells have unequal direction counts ("
                         + ", ".join(f"b={s.bvalue:g}: {s.indices.size}" for s in table)
                         + "); select shells of equal size")
    return np.asarray(b0_idx, dtype=np.int64), tuple(table)


def _sub_scheme(scheme, table, b0_threshold):
    """The selected shells' gradient table, renumbered 0.. in channel order (fitting.py:322-339)."""
    if scheme is None:
        return None
    keep = np.concatenate([s.indices for s in table])
    starts = np.cumsum([0] + [s.indices.size for s in table[:-1]])
    return dwio.GradientScheme(scheme.directions[keep], scheme.bvals[keep], np.zeros(0, np.int64),
                               tuple(dwio.Shell(s.bvalue, np.arange(o, o + s.indices.size))
                                     for o, s in zip(starts, table)), b0_threshold)


def _run(raw_dev: torch.Tensor, code: int, shape3, strides4, slope: float, inter: float, b0_idx, sel, device):
    X, Y, Z = shape3
    lib = _lib.load()
    b0_t = torch.as_tensor(b0_idx, dtype=torch.int64).to(device)
    sel_t = torch.as_tensor(sel, dtype=torch.int64).to(device)
    out = torch.empty((1, len(sel), X, Y, Z), dtype=torch.float32, device=device)
    mask = torch.empty((X, Y, Z), dtype=torch.uint8, device=device)
    ws = torch.empty(int(lib.dl_normalize_b0_workspace_bytes(X, Y, Z)), dtype=torch.uint8, device=device)
    sx, sy, sz, sv = (int(s) for s in strides4)
    _lib.call("dl_normalize_b0_f32", _p(raw_dev), int(code), X, Y, Z, sx, sy, sz, sv, ctypes.c_double(slope),
              ctypes.c_double(inter), _p(b0_t), len(b0_idx), _p(sel_t), len(sel), _p(out), _p(mask), _p(ws),
              _stream())
    return out, mask.bool()


def normalize_b0(raw, bvals_or_scheme, b0_threshold: float = dwio.B0_THRESHOLD,
                 tolerance: float = dwio.SHELL_TOLERANCE, shells: Sequence[float] | None = None, device=None):
    """Divide the diffusion-weighted volumes by the mean b0 volume (fitting.py:253-342), on the GPU.

    raw: (X, Y, Z, V) numpy array or tensor (uint8 / int16 / int32 / float32 / float64, any strides), or a
    dwio.NiftiRaw.  Returns (DwiVolume (1, shells*m, X, Y, Z) fp32 CUDA, excluded (X, Y, Z) bool CUDA).
    """
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    slope, inter = 0.0, 0.0
    if isinstance(raw, dwio.NiftiRaw):
        if len(raw.shape) != 4:
            raise ShapeError(f"raw acquisition must be 4-D, got shape {raw.shape}")
        shape4, code = raw.shape, raw.dtype_code
        strides = raw.strides()
        if raw.scaled:
            slope, inter = raw.slope, raw.inter
        src = np.ascontiguousarray(raw.data)
        host = torch.empty(src.shape, dtype=_TORCH_OF[src.dtype.type], pin_memory=torch.cuda.is_available())
        host.numpy()[...] = src                       # the file's bytes, staged once in pinned memory
        t = host.to(dev, non_blocking=True)
    else:
        t = raw if isinstance(raw, torch.Tensor) else torch.from_numpy(np.asarray(raw))
        if t.dim() != 4:
            raise ShapeError(f"raw acquisition must be 4-D, got shape {tuple(t.shape)}")
        if t.dtype not in _CODE_OF_TORCH:
            t = t.to(torch.float64)
        shape4, code, strides = tuple(t.shape), _CODE_OF_TORCH[t.dtype], t.stride()
        t = t.to(dev)
        strides = t.stride()
    b0_idx, table = select_volumes(bvals_or_scheme, int(shape4[3]), b0_threshold, tolerance, shells)
    sel = np.concatenate([s.indices for s in table]).astype(np.int64)
    out, mask = _run(t, code, shape4[:3], strides, slope, inter, b0_idx, sel, dev)
    scheme = bvals_or_scheme if isinstance(bvals_or_scheme, dwio.GradientScheme) else None
    vol = DwiVolume(out, len(table), check_finite=False, scheme=_sub_scheme(scheme, table, b0_threshold))
    return vol, mask


def load_dwi(nifti_path: str, bvals_path: str, bvecs_path: str, shells: Sequence[float] | None = None,
             b0_threshold: float = dwio.B0_THRESHOLD, tolerance: float = dwio.SHELL_TOLERANCE, device=None):
    """NIfTI + FSL gradient files -> (DwiVolume on the device, excluded mask, selected GradientScheme)."""
    scheme = dwio.read_bvals_bvecs(bvals_path, bvecs_path, b0_threshold=b0_threshold, tolerance=tolerance)
    vol, mask = normalize_b0(dwio.read_nifti_raw(nifti_path), scheme, b0_threshold, tolerance, shells, device)
    return vol, mask, vol.scheme


def _stage_raw(raw, dev):
    """(device tensor of the stored elements, NIfTI code, (X, Y, Z, V), strides, slope, inter)."""
    slope, inter = 0.0, 0.0
    if isinstance(raw, dwio.NiftiRaw):
        if len(raw.shape) != 4:
            raise ShapeError(f"raw acquisition must be 4-D, got shape {raw.shape}")
        if raw.scaled:
            slope, inter = raw.slope, raw.inter
        src = np.ascontiguousarray(raw.data)
        host = torch.empty(src.shape, dtype=_TORCH_OF[src.dtype.type], pin_memory=torch.cuda.is_available())
        host.numpy()[...] = src
        return host.to(dev, non_blocking=True), raw.dtype_code, tuple(raw.shape), raw.strides(), slope, inter
    t = raw if isinstance(raw, torch.Tensor) else torch.from_numpy(np.asarray(raw))
    if t.dim() != 4:
        raise ShapeError(f"raw acquisition must be 4-D, got shape {tuple(t.shape)}")
    if t.dtype not in _CODE_OF_TORCH:
        t = t.to(torch.float64)
    t = t.to(dev)
    return t, _CODE_OF_TORCH[t.dtype], tuple(t.shape), t.stride(), slope, inter


def chain_from_raw(chain, raw, bvals_or_scheme, b0_threshold: float = dwio.B0_THRESHOLD,
                   tolerance: float = dwio.SHELL_TOLERANCE, shells: Sequence[float] | None = None, device=None):
    """chain(normalize_b0(raw)) in one pass over the acquisition (fitting.py:253-342 then the chain).

    chain: a SphericalChain whose Signal2SH matches the selected shells (its per-shell or shared tables are the
    caller's; channel c = shell s, direction i reads stored volume shell[s].indices[i]).  raw: dwio.NiftiRaw or an
    (X, Y, Z, V) array / tensor.  Returns (y, excluded, sub-scheme): y the chain output as a (1, C, X, Y, Z)
    float32 CUDA tensor, excluded the (X, Y, Z) bool mask.  When the acquisition is int16 / float32 in the
    x-fastest layout with volumes contiguous (a NIfTI file's bytes) and the chain fits the fused plan, the
    normalisation runs inside the chain kernel (dl_chain_fwd_raw_f32) and y is a view in the stored voxel order;
    otherwise normalize_b0 then chain (two passes, y C-contiguous).  Forward only (no autograd).
    """
    from . import ops

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    t, code, shape4, strides, slope, inter = _stage_raw(raw, dev)
    X, Y, Z, V = (int(e) for e in shape4)
    b0_idx, table = select_volumes(bvals_or_scheme, V, b0_threshold, tolerance, shells)
    scheme = bvals_or_scheme if isinstance(bvals_or_scheme, dwio.GradientScheme) else None
    sub = _sub_scheme(scheme, table, b0_threshold)
    sel = np.concatenate([s_.indices for s_ in table]).astype(np.int64)
    layers = chain._layers
    first, last = layers[0], layers[-1]
    s_in, n = len(table), int(table[0].indices.size)
    nvox = X * Y * Z
    fused = (code in (4, 16) and tuple(int(a) for a in strides) == (1, X, X * Y, nvox) and nvox % 2 == 0
             and s_in == first.shells_in and n == chain.s2sh.n_gradients and chain.fused())
    if not fused:
        vol, mask = normalize_b0(raw, bvals_or_scheme, b0_threshold, tolerance, shells, dev)
        with torch.no_grad():
            return chain(vol.data), mask, sub
    lib = _lib.load()
    b0_t = torch.as_tensor(b0_idx, dtype=torch.int64).to(dev)
    va = torch.empty(nvox, dtype=torch.float32, device=dev)
    vb = torch.empty(nvox, dtype=torch.float32, device=dev)
    ex = torch.empty(nvox, dtype=torch.uint8, device=dev)
    ws = torch.empty(int(lib.dl_normalize_b0_workspace_bytes(X, Y, Z)), dtype=torch.uint8, device=dev)
    sx, sy, sz, sv = (int(a) for a in strides)
    _lib.call("dl_b0_voxel_scale_f32", _p(t), int(code), X, Y, Z, sx, sy, sz, sv, ctypes.c_double(slope),
              ctypes.c_double(inter), _p(b0_t), len(b0_idx), _p(va), _p(vb), _p(ex), _p(ws), _stream())
    with torch.no_grad():
        args = []
        for layer in layers:
            w, b = layer.sconv.weight, layer.sconv.bias
            args.append((w.reshape(w.shape[0], w.shape[1], w.shape[3]).float().contiguous(),
                         None if b is None else b.float().contiguous(), layer.fold, layer.beta))
        _, _, L, bvec = ops._fold_layers(args)
    s_out, r_in, r_out = last.shells_out, first.r_in, last.r_out
    n_out = chain.sh2s.n_gradients
    sel_t = torch.as_tensor(sel, dtype=torch.int32).to(dev)
    y = torch.empty((s_out * n_out, Z, Y, X), dtype=torch.float32, device=dev)
    wsc = torch.empty(int(lib.dl_chain_workspace_bytes(1, s_in, s_out, n, r_in, r_out, n_out, nvox)),
                      dtype=torch.uint8, device=dev)
    sf, _ = chain.range_state(dev)   # the fp16 pass's scale history (the same signal distribution as chain(x))
    _lib.call("dl_chain_fwd_raw_f32", _p(t), int(code), sv, _p(sel_t), _p(va), _p(vb), _p(y),
              _p(chain.s2sh.fit_matrix), int(chain.s2sh.per_shell), _p(L), _p(bvec), _p(chain.sh2s.basis), _p(wsc),
              _p(sf), s_in, s_out, n, r_in, r_out, n_out, nvox, _stream())
    mask = ex.view(Z, Y, X).permute(2, 1, 0).bool()
    return y.permute(0, 3, 2, 1).unsqueeze(0), mask, sub
