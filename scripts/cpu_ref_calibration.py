"""Calibrate the timed CPU arm (oracle/cpu_baseline.py, the float64 port) against the REAL reference.

Runs only where /root/reference is mounted (the builder container; the GPU box has no reference).  On the same
65,536-voxel cfg4 sample it times, in both of the reference's threading modes (sphdwi bench.py:83-91,
191-208: threads=1 with OpenBLAS threading, and threads=ncores inside threadpool_limits(1)):

  * sphdwi's own forward chain: signal_to_sh -> lsc_forward -> sh_to_signal (fitting.py:206-250, lsc.py:158-199)
  * the port's forward chain (oracle/port.py), and the port's fwd + adjoint step that bench.py times

and checks the two forwards agree.  Writes profiles/r02_cpu_calibration.json.
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba python scripts/cpu_ref_calibration.py
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from oracle import cpu_baseline as cb  # noqa: E402
from oracle import port  # noqa: E402


def med(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def main(nvox=65536):
    import sphdwi
    from sphdwi import fitting, lsc
    from threadpoolctl import threadpool_limits

    from paper_1808_01517_b200.directions import unit_sphere_directions

    dirs = unit_sphere_directions(90)
    x, dy = cb.synthetic_sample(dirs, nvox)
    w = np.random.default_rng(1).normal(size=(3, 3, 6)) / 18.0
    b = np.random.default_rng(1).normal(size=3) * 0.1
    op = fitting.make_fit_operator(dirs, 8, 0.006)
    geom = lsc.build_lsc_geometry(dirs, [5], np.pi / 5, 8, 8, 0.006)
    kern = lsc.LscKernel(weights=w, bias=b)
    vol = fitting.DwiVolume(data=x.reshape(1, 270, nvox, 1, 1), shells=3)
    cores = cb.host_cores()

    def ref_fwd(threads):
        sh = fitting.signal_to_sh(vol, op, threads=threads)
        u = lsc.lsc_forward(sh, kern, geom, threads=threads)
        return fitting.sh_to_signal(u, dirs, threads=threads).data

    orc = cb.ChainOracle(dirs)

    def port_fwd(threads):
        def run(lo, hi):
            xs = x[..., lo:hi, None, None]
            return port.chain_forward(xs, orc.M, orc.geo, w, b, orc.Bt, 3)
        return cb._run_spans(run, nvox, threads)

    y_ref = ref_fwd(1)
    y_port = port.chain_forward(x[..., None, None], orc.M, orc.geo, w, b, orc.Bt, 3)
    agree = port.rel_err(y_port.reshape(y_ref.shape), y_ref)
    out = {"voxels": nvox, "cores": cores, "sphdwi": sphdwi.__version__, "forward_rel_err_port_vs_sphdwi": agree,
           "seconds": {}}
    for mode, threads, limit in (("threads=1+blas", 1, None), (f"threads={cores}+blas1", cores, 1)):
        if limit:
            with threadpool_limits(limit):
                t_ref = med(lambda: ref_fwd(threads))
                t_port = med(lambda: port_fwd(threads))
        else:
            t_ref = med(lambda: ref_fwd(threads))
            t_port = med(lambda: port_fwd(threads))
        t_step = med(lambda: orc.fwd_bwd(x, dy, w, b, threads))
        out["seconds"][mode] = {"sphdwi_forward": t_ref, "port_forward": t_port, "port_fwd_bwd": t_step,
                                "port_over_sphdwi_forward": t_port / t_ref}
    best_ref = min(v["sphdwi_forward"] for v in out["seconds"].values())
    best_port = min(v["port_forward"] for v in out["seconds"].values())
    out["best_forward_voxels_per_s"] = {"sphdwi": nvox / best_ref, "port": nvox / best_port}
    print(json.dumps(out, indent=1))
    with open(os.path.join(ROOT, "profiles", "r02_cpu_calibration.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 65536)
