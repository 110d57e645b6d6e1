"""Timed CPU reference arm: the oracle port of the reference path, on the host's cores.

TEST / BASELINE INFRASTRUCTURE ONLY (bench.py's cpu_baseline and --impl reference legs).

The reference (sphdwi 0.1.0) is pure Python over numpy/OpenBLAS; it cannot travel to the GPU box, so
the timed arm there is this float64 port of the same algorithm (oracle/port.py: resample -> ring
reduce -> refit for the LSC, dgemm per voxel block for the fit / evaluation), timed in the reference's
two threading modes (/root/reference/pkg/src/sphdwi/bench.py:83-91, 191-208):

  (i)  threads=1 in Python, OpenBLAS with its default thread count (one dgemm at a time);
  (ii) threads=ncores voxel spans on a ThreadPool inside threadpool_limits(1) (fitting.py:182-187
       ThreadPool over voxel spans, lsc.py:202-220 _combine_threaded).

The faster mode is reported, with both timings in the sample string.  The backward is the per-stage
adjoint restatement (the reference has no backward); it reuses the forward's SH
coefficients c instead of recomputing them.  scripts/cpu_ref_calibration.py times the real sphdwi
forward beside this port in the builder container (profiles/r02_cpu_calibration.json).
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


def _spans(V: int, threads: int):
    bounds = np.linspace(0, V, threads + 1, dtype=int)
    return [(lo, hi) for lo, hi in zip(bounds[:-1], bounds[1:]) if hi > lo]


def _run_spans(fn, V: int, threads: int):
    """fn(lo, hi) over voxel spans: mode (i) when threads == 1, else mode (ii)."""
    if threads <= 1:
        return [fn(0, V)]
    from threadpoolctl import threadpool_limits

    spans = _spans(V, threads)
    with threadpool_limits(1), ThreadPoolExecutor(max_workers=len(spans)) as pool:
        return list(pool.map(lambda s: fn(*s), spans))


class ChainOracle:
    """Signal2SH(order, dirs, lam) -> LSC(S->S, sizes, alpha, lam) -> SH2Signal(order, dirs), float64."""

    def __init__(self, dirs, order=8, lam=0.006, sizes=(5,), alpha=np.pi / 5, shells=3):
        self.M, _, _ = port.fit_operator(dirs, order, lam)
        self.geo = port.lsc_geometry(dirs, list(sizes), alpha, order, order, lam)
        self.Bt = port.eval_basis(dirs, order)
        self.shells = shells

    def fwd_bwd(self, x, dy, w, b, threads: int | None = None):
        """(y, dx, dW, db); x, dy: (B, S*N, V) float64.  One forward (c kept), one adjoint."""
        threads = threads or host_cores()
        S = self.shells
        so = np.asarray(w).shape[0]
        y = np.empty(x.shape[:1] + (so * self.Bt.shape[0],) + x.shape[2:])
        dx = np.empty_like(x)

        def run(lo, hi):
            xs = x[..., lo:hi, None, None]
            c = port.signal_to_sh(xs, self.M, S)
            u = port.lsc_forward(c, w, b, self.geo)
            y[..., lo:hi] = port.sh_to_signal(u, self.Bt, so)[..., 0, 0]
            g = port.sh_to_signal_adjoint(dy[..., lo:hi, None, None], self.Bt, so)
            dc, gW, gb = port.lsc_backward(c, g, w, self.geo)
            dx[..., lo:hi] = port.signal_to_sh_adjoint(dc, self.M, S)[..., 0, 0]
            return gW, gb

        parts = _run_spans(run, x.shape[-1], threads)
        return y, dx, sum(p[0] for p in parts), sum(p[1] for p in parts)

    def round_trip(self, x, dy, threads: int | None = None):
        """cfg2: y = B' M x and dx = M^T B'^T dy per shell."""
        threads = threads or host_cores()
        S = self.shells
        y = np.empty_like(x)
        dx = np.empty_like(x)

        def run(lo, hi):
            xs = x[..., lo:hi, None, None]
            y[..., lo:hi] = port.sh_to_signal(port.signal_to_sh(xs, self.M, S), self.Bt, S)[..., 0, 0]
            g = port.sh_to_signal_adjoint(dy[..., lo:hi, None, None], self.Bt, S)
            dx[..., lo:hi] = port.signal_to_sh_adjoint(g, self.M, S)[..., 0, 0]

        _run_spans(run, x.shape[-1], threads)
        return y, dx

    def signal_to_sh(self, x, threads: int | None = None):
        """cfg1: c = M x (S = 1)."""
        threads = threads or host_cores()
        c = np.empty(x.shape[:1] + (self.M.shape[0] * self.shells,) + x.shape[2:])

        def run(lo, hi):
            c[..., lo:hi] = port.signal_to_sh(x[..., lo:hi, None, None], self.M, self.shells)[..., 0, 0]

        _run_spans(run, x.shape[-1], threads)
        return c

    def lsc_fwd_bwd(self, c, g, w, b, threads: int | None = None):
        """cfg3: LSC forward and its adjoint on SH volumes (B, S*R, V)."""
        threads = threads or host_cores()
        so = np.asarray(w).shape[0]
        u = np.empty(c.shape[:1] + (so * self.geo["refit"].shape[0],) + c.shape[2:])
        dc = np.empty_like(c)

        def run(lo, hi):
            cs = c[..., lo:hi, None, None]
            u[..., lo:hi] = port.lsc_forward(cs, w, b, self.geo)[..., 0, 0]
            d, gW, gb = port.lsc_backward(cs, g[..., lo:hi, None, None], w, self.geo)
            dc[..., lo:hi] = d[..., 0, 0]
            return gW, gb

        parts = _run_spans(run, c.shape[-1], threads)
        return u, dc, sum(p[0] for p in parts), sum(p[1] for p in parts)


    def train_step(self, x, t, layers, threads: int | None = None):
        """cfg5: Signal2SH -> LSC_1 -> ... -> LSC_n -> SH2Signal, MSE against t, every layer's (dW, db)."""
        threads = threads or host_cores()
        S = self.shells
        count = float(t.size)

        def run(lo, hi):
            us = [port.signal_to_sh(x[..., lo:hi, None, None], self.M, S)]
            for w, b in layers:
                us.append(port.lsc_forward(us[-1], w, b, self.geo))
            y = port.sh_to_signal(us[-1], self.Bt, np.asarray(layers[-1][0]).shape[0])
            r = y - t[..., lo:hi, None, None]
            g = port.sh_to_signal_adjoint(2.0 * r / count, self.Bt, np.asarray(layers[-1][0]).shape[0])
            grads = []
            for k in reversed(range(len(layers))):
                g, gW, gb = port.lsc_backward(us[k], g, layers[k][0], self.geo)
                grads.append((gW, gb))
            return float(np.sum(r * r)), grads[::-1]

        parts = _run_spans(run, x.shape[-1], threads)
        loss = sum(p[0] for p in parts) / count
        grads = [(sum(p[1][k][0] for p in parts), sum(p[1][k][1] for p in parts)) for k in range(len(layers))]
        return loss, grads


def synthetic_sample(dirs, nvox: int, shells: int = 3, order: int = 8, seed: int = 0, batch: int = 1):
    """Band-limited signals B c + N(0, 0.02^2) (phantom.py:77-88), upstream grad N(0,1); fp32-exact f64."""
    B = port.eval_basis(dirs, order)
    out = []
    for b in range(batch):
        xs = [B @ port.bandlimited_coeffs(np.random.default_rng(1000 + s + seed + 31 * b), order, nvox)
              for s in range(shells)]
        out.append(np.concatenate(xs, axis=0))
    x = np.stack(out) + np.random.default_rng(7 + seed).normal(0, 0.02, size=(batch, shells * B.shape[0], nvox))
    dy = np.random.default_rng(2 + seed).normal(size=x.shape)
    return x.astype(np.float32).astype(np.float64), dy.astype(np.float32).astype(np.float64)


def time_modes(fn, repeats: int = 3, warm=None):
    """Median seconds of fn(threads) in both threading modes; returns (best_s, best_threads, {mode: s})."""
    cores = host_cores()
    res = {}
    for mode, threads in (("threads=1+blas", 1), (f"threads={cores}+blas1", cores)):
        (warm or fn)(threads)
        ts = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            fn(threads)
            ts.append(time.perf_counter() - t0)
        res[mode] = (float(np.median(ts)), threads)
    best = min(res.items(), key=lambda kv: kv[1][0])
    return best[1][0], best[1][1], {k: v[0] for k, v in res.items()}, best[0]


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        return max((i.get("num_threads") or 1) for i in threadpool_info() if i.get("user_api") == "blas")
    except Exception:  # pragma: no cover
        return 1
