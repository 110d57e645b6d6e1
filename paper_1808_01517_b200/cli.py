"""Command line: the reference CLI's transform commands on the GPU path.

    python -m paper_1808_01517_b200 signal2sh | sh2signal | lsc | chain | bench ...

Same arguments, outputs and exit codes as the reference (cli.py:48-341): 0 success, 2 usage/validation,
3 numerical failure, 4 I/O failure; diagnostics on stderr; outputs written atomically (dwio.write_nifti).
signal2sh reads the acquisition through the fused ingest kernel (ingest.load_dwi); `chain` is new: the fused
Signal2SH -> LSC -> SH2Signal of one command.  `bench` prints the reference's CSV schema
(direction,order,voxels,method,seconds,max_dev; bench.py:40) with method "gpu" (device-resident, CUDA
events) and "gpu-e2e" (host arrays in and out), max_dev against a float64 numpy product of the same operator.
The reference's `phantom` command is out of scope here (not on the path).
"""

from __future__ import annotations

import argparse
import math
import os
import sys
import tempfile

import numpy as np
import torch

from . import dwio, functional as F, ingest, kernel_io
from .errors import (GradientParseError, IllPosedFitError, KernelMismatchError, MissingB0Error, NiftiError,
                     ShapeError, SphdwiError)
from .geometry import (ShBasisSpec, as_unit_directions, build_lsc_geometry, coeff_count, eval_basis,
                       high_degree_energy_fraction, make_fit_operator, make_moving_average_kernel)

EXIT_VALIDATION, EXIT_NUMERICAL, EXIT_IO = 2, 3, 4
_ORDER_OF_R = {coeff_count(o): o for o in range(0, 17, 2)}
CSV_HEADER = "direction,order,voxels,method,seconds,max_dev"


def _say(msg: str) -> None:
    print(msg, file=sys.stderr)


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1808_01517_b200",
                                 description="Spherical-harmonic transforms and local spherical convolution for "
                                             "diffusion-MRI volumes on B200 (sm_100a).")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("signal2sh", help="b0-normalise a DWI volume and fit SH coefficients")
    p.add_argument("--dwi", required=True)
    p.add_argument("--bvals", required=True)
    p.add_argument("--bvecs", required=True)
    p.add_argument("--order", type=int, default=4)
    p.add_argument("--lambda", dest="lb_lambda", type=float, default=0.006)
    p.add_argument("--shell", type=float, action="append")
    p.add_argument("--threads", type=int, default=1, help="accepted for compatibility")
    p.add_argument("--out", required=True)
    p = sub.add_parser("sh2signal", help="evaluate SH coefficients at target directions")
    p.add_argument("--sh", required=True)
    p.add_argument("--dirs")
    p.add_argument("--bvals")
    p.add_argument("--bvecs")
    p.add_argument("--shell", type=float, action="append")
    p.add_argument("--order", type=int, default=4)
    p.add_argument("--threads", type=int, default=1)
    p.add_argument("--out", required=True)
    p = sub.add_parser("lsc", help="local spherical convolution of an SH volume")
    p.add_argument("--sh", required=True)
    p.add_argument("--bvals", required=True)
    p.add_argument("--bvecs", required=True)
    p.add_argument("--shell", type=float, action="append")
    p.add_argument("--kernel")
    p.add_argument("--moving-average", metavar="N,ALPHA")
    p.add_argument("--order-out", type=int)
    p.add_argument("--lambda", dest="lb_lambda", type=float, default=0.006)
    p.add_argument("--threads", type=int, default=1)
    p.add_argument("--out", required=True)
    p = sub.add_parser("chain", help="fused Signal2SH -> LSC -> SH2Signal of a DWI volume")
    p.add_argument("--dwi", required=True)
    p.add_argument("--bvals", required=True)
    p.add_argument("--bvecs", required=True)
    p.add_argument("--shell", type=float, action="append")
    p.add_argument("--order", type=int, default=8)
    p.add_argument("--lambda", dest="lb_lambda", type=float, default=0.006)
    p.add_argument("--kernel")
    p.add_argument("--moving-average", metavar="N,ALPHA")
    p.add_argument("--out", required=True)
    p = sub.add_parser("bench", help="GPU transform benchmark (reference CSV schema)")
    p.add_argument("--orders", default="2,4,6,8")
    p.add_argument("--voxels", type=int, default=450_000)
    p.add_argument("--repeats", type=int, default=3)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--dirs", type=int, default=90, choices=(30, 60, 90))
    p.add_argument("--lambda", dest="lb_lambda", type=float, default=0.006)
    p.add_argument("--out")
    return ap


# --------------------------------------------------------------------------- helpers
def _to_nifti(data5: torch.Tensor, path: str, affine) -> None:
    """(1, C, X, Y, Z) device tensor -> (X, Y, Z, C) float32 NIfTI (cli.py:154-156)."""
    dwio.write_nifti(path, np.moveaxis(data5[0].detach().cpu().numpy(), 0, 3), affine=affine, dtype=np.float32)


def _load_sh(path: str, order: int | None, shells: int | None = None):
    """SH NIfTI -> (ShVolume on the device, affine); order / shell count inferred as in cli.py:120-151."""
    data, affine, _ = dwio.read_nifti(path)
    if data.ndim != 4:
        raise ShapeError(f"{path}: SH volume must be 4-D, got {data.ndim}-D")
    nvol = data.shape[3]
    if order is not None:
        r = coeff_count(order)
        if shells is None:
            if nvol % r:
                raise ShapeError(f"{path}: {nvol} volumes is not a multiple of R = {r} for order {order} (expects {r})")
            shells = nvol // r
        elif shells * r != nvol:
            raise ShapeError(f"{path}: expected shells ({shells}) * R ({r}) = {shells * r} volumes, found {nvol} "
                             f"(expects {shells * r})")
    else:
        shells = shells or 1
        if nvol % shells or nvol // shells not in _ORDER_OF_R:
            raise ShapeError(f"{path}: cannot infer SH order from {nvol} volumes and {shells} shell(s)")
        order = _ORDER_OF_R[nvol // shells]
    t = torch.tensor(np.moveaxis(data, 3, 0)[None], dtype=torch.float32, device="cuda")
    return F.ShVolume(t, ShBasisSpec(order), shells), affine


def _kernel_from_args(args, n_shells: int):
    if (args.kernel is None) == (args.moving_average is None):
        raise ShapeError("give exactly one of --kernel or --moving-average")
    if args.kernel is not None:
        return kernel_io.load_kernel_json(args.kernel)
    try:
        n, alpha = args.moving_average.split(",")
        sizes, alpha = (int(n),), float(alpha)
    except ValueError:
        raise ShapeError(f"--moving-average expects 'N,ALPHA', got {args.moving_average!r}") from None
    return make_moving_average_kernel(sizes, shells_in=n_shells, shells_out=n_shells), sizes, alpha


def _mean_l2(vol) -> float:
    r = vol.basis_spec.coeff_count
    c = vol.data[0].detach().double().cpu().numpy()
    return float(np.mean([high_degree_energy_fraction(c[s * r:(s + 1) * r], vol.basis_spec.order, axis=0)
                          for s in range(vol.shells)]))


# --------------------------------------------------------------------------- commands
def cmd_signal2sh(a) -> int:
    vol, _, scheme = ingest.load_dwi(a.dwi, a.bvals, a.bvecs, shells=a.shell)
    ops_ = [make_fit_operator(scheme.shell_directions(s.bvalue), a.order, a.lb_lambda) for s in scheme.shells]
    _say(f"R={ops_[0].basis_spec.coeff_count} cond={max(o.cond for o in ops_):.3e}")
    _to_nifti(F.signal_to_sh(vol, ops_).data, a.out, dwio.read_nifti_raw(a.dwi).affine)
    return 0


def cmd_sh2signal(a) -> int:
    if (a.dirs is None) == (a.bvecs is None):
        raise ShapeError("give either --dirs or the --bvals/--bvecs/--shell triple")
    if a.dirs is not None:
        rows = np.asarray(dwio._numeric_rows(a.dirs), dtype=np.float64)
        if rows.ndim != 2 or rows.shape[1] != 3:
            raise GradientParseError(f"{a.dirs}: expected one 'x y z' row per direction")
        dirs = as_unit_directions(rows)
    else:
        if a.bvals is None or not a.shell:
            raise ShapeError("--bvecs needs --bvals and at least one --shell")
        dirs = dwio.read_bvals_bvecs(a.bvals, a.bvecs).shell_directions(a.shell[0])
    sh, affine = _load_sh(a.sh, a.order)
    _to_nifti(F.sh_to_signal(sh, dirs).data, a.out, affine)
    return 0


def _selected_origins(a):
    scheme = dwio.read_bvals_bvecs(a.bvals, a.bvecs)
    chosen = [scheme.shell(b) for b in (a.shell or scheme.shell_bvalues())]
    if not chosen:
        raise ShapeError("no shells selected")
    if len({s.indices.size for s in chosen}) != 1:
        raise ShapeError("selected shells must share one direction count")
    return scheme.directions[chosen[0].indices], len(chosen)


def cmd_lsc(a) -> int:
    if (a.kernel is None) == (a.moving_average is None):
        raise ShapeError("give exactly one of --kernel or --moving-average")
    origins, n_shells = _selected_origins(a)
    kernel, sizes, alpha = _kernel_from_args(a, n_shells)
    if kernel.shells_in != n_shells:
        raise ShapeError(f"kernel expects {kernel.shells_in} input shells, selection has {n_shells}")
    sh, affine = _load_sh(a.sh, None, kernel.shells_in)
    geom = build_lsc_geometry(origins, sizes, alpha, sh.basis_spec.order,
                              a.order_out if a.order_out is not None else sh.basis_spec.order, a.lb_lambda)
    out = F.lsc_forward(sh, kernel, geom)
    _say(f"mean l>=2 energy fraction: {_mean_l2(sh):.4f} -> {_mean_l2(out):.4f}")
    _to_nifti(out.data, a.out, affine)
    return 0


def cmd_chain(a) -> int:
    """normalize_b0 -> signal2sh -> lsc -> sh2signal of one acquisition.  The b0 normalisation runs inside the fused
    chain kernel, which reads the file's stored volumes (ingest.chain_from_raw); the output comes back in the
    file's voxel order, which is also the order the output NIfTI stores."""
    from . import modules as M

    raw = dwio.read_nifti_raw(a.dwi)
    scheme = dwio.read_bvals_bvecs(a.bvals, a.bvecs)
    if len(raw.shape) != 4:
        raise ShapeError(f"raw acquisition must be 4-D, got shape {raw.shape}")
    _, table = ingest.select_volumes(scheme, int(raw.shape[3]), shells=a.shell)
    sub = ingest._sub_scheme(scheme, table, scheme.b0_threshold)
    tables = np.stack([sub.shell_directions(b) for b in sub.shell_bvalues()])
    kernel, sizes, alpha = _kernel_from_args(a, len(table))
    s2sh = M.Signal2SH(a.order, tables, lb_lambda=a.lb_lambda).cuda()
    lsc = M.LocalSphericalConvolution(kernel.shells_in, kernel.shells_out, a.order, a.order, tables[0], sizes,
                                      lb_lambda=a.lb_lambda, angular_distance=alpha).cuda()
    lsc.load_kernel(kernel)
    sh2s = M.SH2Signal(a.order, tables[0]).cuda()
    y, _, _ = ingest.chain_from_raw(M.SphericalChain(s2sh, lsc, sh2s), raw, scheme, shells=a.shell)
    _to_nifti(y, a.out, raw.affine)
    return 0


def cmd_bench(a) -> int:
    from .directions import unit_sphere_directions

    try:
        orders = [int(t) for t in str(a.orders).split(",") if t.strip()]
    except ValueError:
        raise ShapeError(f"--orders expects comma-separated integers, got {a.orders!r}") from None
    dirs = unit_sphere_directions(a.dirs)
    rng = np.random.default_rng(a.seed)
    rows = []
    for order in orders:
        op = make_fit_operator(dirs, order, a.lb_lambda)
        B = eval_basis(dirs, order)
        x = rng.uniform(0.1, 1.2, size=(1, a.dirs, a.voxels, 1, 1)).astype(np.float32)
        xt = torch.tensor(x, device="cuda")
        for direction, run, host_ref in (
                ("signal2sh", lambda v: F.signal_to_sh(F.DwiVolume(v, 1, check_finite=False), op).data,
                 lambda: op.fit_matrix @ x[0, :, :, 0, 0].astype(np.float64)),
                ("sh2signal", lambda v: F.sh_to_signal(F.ShVolume(v, op.basis_spec, 1), dirs).data,
                 lambda: B @ (op.fit_matrix @ x[0, :, :, 0, 0].astype(np.float64)))):
            inp = xt if direction == "signal2sh" else run_prev
            out = run(inp)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            times = []
            for _ in range(max(1, a.repeats)):
                ev0.record()
                out = run(inp)
                ev1.record()
                torch.cuda.synchronize()
                times.append(ev0.elapsed_time(ev1) / 1e3)
            ref = host_ref()
            dev = float(np.max(np.abs(out[0, :, :, 0, 0].double().cpu().numpy() - ref)))
            rows.append(f"{direction},{order},{a.voxels},gpu,{float(np.median(times)):.6f},{dev:.3e}")
            host = inp.cpu().pin_memory()
            times = []
            for _ in range(max(1, a.repeats)):
                ev0.record()
                res = run(host.to("cuda", non_blocking=True)).cpu()
                ev1.record()
                torch.cuda.synchronize()
                times.append(ev0.elapsed_time(ev1) / 1e3)
            rows.append(f"{direction},{order},{a.voxels},gpu-e2e,{float(np.median(times)):.6f},{dev:.3e}")
            run_prev = out if direction == "signal2sh" else None
    text = CSV_HEADER + "\n" + "\n".join(rows) + "\n"
    if a.out:
        folder = os.path.dirname(os.path.abspath(a.out)) or "."
        fd, tmp = tempfile.mkstemp(prefix=".bench-", suffix=".csv", dir=folder)
        with os.fdopen(fd, "w") as fh:
            fh.write(text)
        os.replace(tmp, a.out)
    else:
        sys.stdout.write(text)
    return 0


HANDLERS = {"signal2sh": cmd_signal2sh, "sh2signal": cmd_sh2signal, "lsc": cmd_lsc, "chain": cmd_chain,
            "bench": cmd_bench}


def main(argv=None) -> int:
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        return HANDLERS[args.command](args)
    except (ShapeError, GradientParseError, KernelMismatchError, MissingB0Error, ValueError) as exc:
        _say(f"paper_1808_01517_b200: {exc}")
        return EXIT_VALIDATION
    except IllPosedFitError as exc:
        _say(f"paper_1808_01517_b200: {exc}")
        return EXIT_NUMERICAL
    except (NiftiError, OSError) as exc:
        _say(f"paper_1808_01517_b200: {exc}")
        return EXIT_IO
    except SphdwiError as exc:
        _say(f"paper_1808_01517_b200: {exc}")
        return EXIT_VALIDATION
