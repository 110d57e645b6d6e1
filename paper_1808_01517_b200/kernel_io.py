"""LSC kernel interchange: the reference's JSON document for trained ring kernels.

Same fields, checks and errors as lsc.save_kernel_json / lsc.load_kernel_json (lsc.py:27, 223-277):
{"shells_in", "shells_out", "kernel_sizes", "angular_distance", "weights" (S_out x S_in x K), "bias" (S_out)}.
save_module / load_module move a LocalSphericalConvolution's `.sconv` parameters through that document, so
kernels trained here load in the reference (and the reverse); torch state_dicts keep working as usual.
"""

from __future__ import annotations

import json
import os
import tempfile

import numpy as np

from .errors import KernelMismatchError
from .geometry import LscKernel

KERNEL_JSON_FIELDS = ("shells_in", "shells_out", "kernel_sizes", "angular_distance", "weights", "bias")


def save_kernel_json(path: str, kernel: LscKernel, kernel_sizes, angular_distance: float) -> None:
    """Write `kernel` with its ring layout; the file appears atomically (lsc.py:223-249)."""
    sizes = [int(s) for s in kernel_sizes]
    k_ring = 1 + sum(sizes)
    if kernel.kernel_len != k_ring:
        raise KernelMismatchError(f"kernel length K = {kernel.kernel_len} does not match kernel_sizes K = {k_ring}")
    doc = dict(shells_in=kernel.shells_in, shells_out=kernel.shells_out, kernel_sizes=sizes,
               angular_distance=float(angular_distance), weights=kernel.weights.tolist(), bias=kernel.bias.tolist())
    folder = os.path.dirname(os.path.abspath(path)) or "."
    fd, tmp = tempfile.mkstemp(prefix=".kernel-", suffix=".json", dir=folder)
    try:
        with os.fdopen(fd, "w") as fh:
            fh.write(json.dumps(doc, indent=2) + "\n")
        mask = os.umask(0)
        os.umask(mask)
        os.chmod(tmp, 0o666 & ~mask)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def load_kernel_json(path: str):
    """(LscKernel, kernel_sizes, angular_distance) from a kernel document (lsc.py:252-277)."""
    with open(path) as fh:
        try:
            doc = json.load(fh)
        except json.JSONDecodeError as exc:
            raise KernelMismatchError(f"{path}: not valid JSON ({exc})") from exc
    missing = [f for f in KERNEL_JSON_FIELDS if f not in doc]
    if missing:
        raise KernelMismatchError(f"{path}: missing fields {missing}")
    sizes = tuple(int(s) for s in doc["kernel_sizes"])
    w = np.asarray(doc["weights"], dtype=np.float64)
    b = np.asarray(doc["bias"], dtype=np.float64)
    so, si = int(doc["shells_out"]), int(doc["shells_in"])
    if w.ndim != 3 or w.shape[:2] != (so, si):
        raise KernelMismatchError(f"{path}: weights shape {w.shape} does not match declared shells "
                                  f"({so} out, {si} in)")
    if w.shape[2] != 1 + sum(sizes):
        raise KernelMismatchError(f"{path}: weights length K = {w.shape[2]} does not match kernel_sizes "
                                  f"K = {1 + sum(sizes)}")
    return LscKernel(weights=w, bias=b), sizes, float(doc["angular_distance"])


def save_module(path: str, lsc) -> None:
    """A LocalSphericalConvolution's current parameters as a kernel document."""
    save_kernel_json(path, lsc.kernel, lsc.kernel_sizes, lsc.angular_distance)


def load_module(path: str, lsc) -> None:
    """Load a kernel document into `lsc`; its ring layout must match the module's geometry."""
    kernel, sizes, alpha = load_kernel_json(path)
    if tuple(sizes) != tuple(lsc.kernel_sizes) or not np.isclose(alpha, lsc.angular_distance, rtol=0, atol=1e-12):
        raise KernelMismatchError(f"{path}: ring layout {sizes} at {alpha:g} rad does not match the module's "
                                  f"{tuple(lsc.kernel_sizes)} at {lsc.angular_distance:g} rad")
    lsc.load_kernel(kernel)
