"""Golden files for the ingest path, made by the REAL reference (sphdwi 0.1.0).

Run in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_ingest_golden.py

Writes tests/golden/ingest/:
  acq.nii.gz    int16 acquisition (9 x 7 x 6 voxels, 2 b0 + 2 shells x 6 directions, interleaved), written by
                the reference's dwio.write_nifti, then scl_slope = 0.5 / scl_inter = 10 patched into the header
  acq.bval, acq.bvec   the gradient table (reference dwio.write_bvals_bvecs)
  kernel_ref.json  a 2 -> 3 shell, two-ring LSC kernel written by the reference's lsc.save_kernel_json
  cli_sh.nii.gz, cli_lsc.nii.gz, cli_sig.nii.gz  the reference CLI's signal2sh (order 4) / lsc (moving
                average 5 at pi/5) / sh2signal (shell 1000 directions) outputs on acq.nii.gz
  cli_lsc_k.nii.gz  the reference CLI's lsc with kernel_ref.json (2 -> 3 shells, rings [5, 7]) to order 2
  expected.npz  reference outputs: read_nifti data (float64, slope applied), normalize_b0 on the file's data
                (all shells; shell 2000 only) with the exclusion mask, and normalize_b0 of an in-memory float64
                array with a zero-b0 voxel.
Nothing here is imported by the product; tests read the files.
"""

from __future__ import annotations

import gzip
import os
import struct
import sys

import numpy as np

sys.path.insert(0, os.environ.get("SPHDWI_REF", "/root/reference/pkg/src"))
from sphdwi import dwio  # noqa: E402
from sphdwi.fitting import normalize_b0  # noqa: E402
from sphdwi.lsc import LscKernel, save_kernel_json  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ingest")


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(7)
    X, Y, Z = 9, 7, 6
    bvals = np.array([0, 1000, 2000, 1000, 5, 2000, 1000, 2000, 1000, 2000, 1000, 2000, 1000, 2000], float)
    dirs = rng.normal(size=(bvals.size, 3))
    dirs[bvals <= 50] = 0.0
    dwio.write_bvals_bvecs(bvals, dirs, os.path.join(OUT, "acq.bval"), os.path.join(OUT, "acq.bvec"))
    stored = rng.integers(200, 3000, size=(X, Y, Z, bvals.size)).astype(np.int16)
    stored[..., bvals <= 50] = rng.integers(2500, 4000, size=(X, Y, Z, 2)).astype(np.int16)
    stored[0, 0, 0, bvals <= 50] = -20       # b0 mean <= eps after scaling -> excluded voxel
    path = os.path.join(OUT, "acq.nii.gz")
    dwio.write_nifti(path, stored, affine=np.diag([1.25, 1.25, 1.25, 1.0]), dtype=np.int16)
    with gzip.open(path, "rb") as fh:
        raw = bytearray(fh.read())
    struct.pack_into("<ff", raw, 112, 0.5, 10.0)   # scl_slope, scl_inter
    with gzip.open(path, "wb") as fh:
        fh.write(bytes(raw))
    data, affine, _ = dwio.read_nifti(path)
    scheme = dwio.read_bvals_bvecs(os.path.join(OUT, "acq.bval"), os.path.join(OUT, "acq.bvec"))
    vol, mask = normalize_b0(data, scheme)
    vol2, mask2 = normalize_b0(data, scheme, shells=[2000.0])
    mem = rng.uniform(0.5, 2.0, size=(5, 4, 3, 7)) * 800.0
    mem[1, 2, 0, 0] = 0.0
    mem[1, 2, 0, 1] = 0.0
    vol3, mask3 = normalize_b0(mem, [0.0, 0.0, 1000.0, 1000.0, 1000.0, 2000.0, 2000.0], shells=[1000.0])
    np.savez_compressed(os.path.join(OUT, "expected.npz"), data=data, affine=affine, vol=vol.data, mask=mask,
                        vol_b2000=vol2.data, mask_b2000=mask2, mem=mem, vol_mem=vol3.data, mask_mem=mask3,
                        sub_bvals=vol.scheme.bvals, sub_dirs=vol.scheme.directions)
    kw = rng.normal(size=(3, 2, 1 + 5 + 7))
    save_kernel_json(os.path.join(OUT, "kernel_ref.json"), LscKernel(weights=kw, bias=rng.normal(size=3)), [5, 7],
                     np.pi / 8)
    from sphdwi.cli import main as cli
    j = lambda n: os.path.join(OUT, n)  # noqa: E731
    g = ["--bvals", j("acq.bval"), "--bvecs", j("acq.bvec")]
    assert cli(["signal2sh", "--dwi", j("acq.nii.gz"), *g, "--order", "4", "--out", j("cli_sh.nii.gz")]) == 0
    assert cli(["lsc", "--sh", j("cli_sh.nii.gz"), *g, "--moving-average", "5,0.6283185307",
                "--out", j("cli_lsc.nii.gz")]) == 0
    assert cli(["sh2signal", "--sh", j("cli_lsc.nii.gz"), *g, "--shell", "1000", "--order", "4",
                "--out", j("cli_sig.nii.gz")]) == 0
    assert cli(["lsc", "--sh", j("cli_sh.nii.gz"), *g, "--kernel", j("kernel_ref.json"), "--order-out", "2",
                "--out", j("cli_lsc_k.nii.gz")]) == 0
    print("wrote", OUT, vol.data.shape, int(mask.sum()), vol3.data.shape, int(mask3.sum()))


if __name__ == "__main__":
    main()
