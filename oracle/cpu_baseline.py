"""Timed CPU reference arm: the oracle port of the reference path, on all host cores.

TEST / BASELINE INFRASTRUCTURE ONLY (bench.py's cpu_baseline and --impl reference legs).

Mirrors the reference's own parallel mode (threads = ncores inside
threadpool_limits(1): fitting.py:182-187 ThreadPool over voxel spans,
lsc.py:202-220 _combine_threaded), i.e. float64 numpy/BLAS per voxel span, one
span per thread.  The backward is the per-stage adjoint restatement
(port.chain_backward) -- the reference has no backward.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import port


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class ChainOracle:
    """Signal2SH(8, dirs, lam) -> LSC(S->S, [5], pi/5, lam) -> SH2Signal(8, dirs), float64."""

    def __init__(self, dirs, order=8, lam=0.006, sizes=(5,), alpha=np.pi / 5, shells=3):
        self.M, _, _ = port.fit_operator(dirs, order, lam)
        self.geo = port.lsc_geometry(dirs, list(sizes), alpha, order, order, lam)
        self.Bt = port.eval_basis(dirs, order)
        self.shells = shells

    def fwd_bwd(self, x, dy, w, b, threads: int | None = None):
        """(y, dx, dW, db) over voxel spans in parallel; x, dy: (B, S*N, V) float64."""
        threads = threads or host_cores()
        V = x.shape[-1]
        bounds = np.linspace(0, V, threads + 1, dtype=int)
        spans = [(lo, hi) for lo, hi in zip(bounds[:-1], bounds[1:]) if hi > lo]
        y = np.empty_like(x)
        dx = np.empty_like(x)

        def run(span):
            lo, hi = span
            xs = x[..., lo:hi, None, None]
            ds = dy[..., lo:hi, None, None]
            y[..., lo:hi] = port.chain_forward(xs, self.M, self.geo, w, b, self.Bt, self.shells)[..., 0, 0]
            gx, gW, gb = port.chain_backward(xs, ds, self.M, self.geo, w, self.Bt, self.shells)
            dx[..., lo:hi] = gx[..., 0, 0]
            return gW, gb

        from threadpoolctl import threadpool_limits

        with threadpool_limits(1), ThreadPoolExecutor(max_workers=len(spans)) as pool:
            parts = list(pool.map(run, spans))
        dW = sum(p[0] for p in parts)
        db = sum(p[1] for p in parts)
        return y, dx, dW, db


def synthetic_sample(dirs, nvox: int, shells: int = 3, order: int = 8, seed: int = 0):
    """Band-limited signals B c + N(0, 0.02^2) (phantom.py:77-88), upstream grad N(0,1); fp32-exact f64."""
    B = port.eval_basis(dirs, order)
    xs = [B @ port.bandlimited_coeffs(np.random.default_rng(1000 + s + seed), order, nvox) for s in range(shells)]
    x = np.concatenate(xs, axis=0)[None] + np.random.default_rng(7 + seed).normal(0, 0.02, size=(1, shells * B.shape[0], nvox))
    dy = np.random.default_rng(2 + seed).normal(size=x.shape)
    return x.astype(np.float32).astype(np.float64), dy.astype(np.float32).astype(np.float64)


def time_fwd_bwd(dirs, nvox: int, repeats: int = 3, threads: int | None = None, w=None, b=None):
    """Median seconds of the oracle chain fwd+bwd on `nvox` voxels (one warm-up, as bench.py:180-208)."""
    threads = threads or host_cores()
    orc = ChainOracle(dirs)
    x, dy = synthetic_sample(dirs, nvox)
    if w is None:
        w = np.random.default_rng(1).normal(size=(3, 3, 6)) / 18.0
        b = np.random.default_rng(1).normal(size=3) * 0.1
    orc.fwd_bwd(x[..., : min(nvox, 4096)], dy[..., : min(nvox, 4096)], w, b, threads)
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        orc.fwd_bwd(x, dy, w, b, threads)
        times.append(time.perf_counter() - t0)
    return float(np.median(times)), threads
