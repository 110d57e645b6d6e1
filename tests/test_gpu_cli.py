"""The CLI (cli.py) against the reference CLI's own outputs on the same files (tests/golden/ingest/cli_*.nii.gz,
made by tests/golden/make_ingest_golden.py): signal2sh, lsc, sh2signal, and the fused `chain` command, which
must equal the reference's three commands composed.  Tolerances as the parity suite: 1e-5 for SH coefficients
and signals, 1e-4 after the LSC (normwise max relative error)."""

import os

import numpy as np
import pytest
import torch

from conftest import ROOT
from oracle import port
from paper_1808_01517_b200 import dwio
from paper_1808_01517_b200.cli import main

pytestmark = pytest.mark.gpu
G = os.path.join(ROOT, "tests", "golden", "ingest")


@pytest.fixture(scope="module", autouse=True)
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1808_01517_b200._build import build_library

    build_library()


def j(n):
    return os.path.join(G, n)


GR = ["--bvals", j("acq.bval"), "--bvecs", j("acq.bvec")]


def rd(p):
    return dwio.read_nifti(p)[0]


def test_cli_commands_match_reference(tmp_path):
    sh = str(tmp_path / "sh.nii.gz")
    assert main(["signal2sh", "--dwi", j("acq.nii.gz"), *GR, "--order", "4", "--out", sh]) == 0
    assert port.rel_err(rd(sh), rd(j("cli_sh.nii.gz"))) <= 1e-5
    ls = str(tmp_path / "lsc.nii.gz")
    assert main(["lsc", "--sh", j("cli_sh.nii.gz"), *GR, "--moving-average", "5,0.6283185307", "--out", ls]) == 0
    assert port.rel_err(rd(ls), rd(j("cli_lsc.nii.gz"))) <= 1e-4
    sg = str(tmp_path / "sig.nii.gz")
    assert main(["sh2signal", "--sh", j("cli_lsc.nii.gz"), *GR, "--shell", "1000", "--order", "4", "--out", sg]) == 0
    assert port.rel_err(rd(sg), rd(j("cli_sig.nii.gz"))) <= 1e-5


def test_cli_chain_equals_reference_composition(tmp_path):
    out = str(tmp_path / "chain.nii.gz")
    assert main(["chain", "--dwi", j("acq.nii.gz"), *GR, "--order", "4", "--moving-average", "5,0.6283185307",
                 "--out", out]) == 0
    assert port.rel_err(rd(out), rd(j("cli_sig.nii.gz"))) <= 1e-4


def test_cli_exit_codes(tmp_path):
    o = str(tmp_path / "o.nii")
    assert main(["lsc", "--sh", j("cli_sh.nii.gz"), *GR, "--out", o]) == 2                       # no kernel
    assert main(["signal2sh", "--dwi", str(tmp_path / "missing.nii"), *GR, "--out", o]) == 4     # I/O
    assert main(["signal2sh", "--dwi", j("acq.nii.gz"), *GR, "--shell", "3000", "--out", o]) == 2
    assert main(["signal2sh", "--dwi", j("acq.nii.gz"), *GR, "--order", "8", "--lambda", "0", "--out", o]) == 3


def test_cli_bench_csv(tmp_path):
    p = str(tmp_path / "b.csv")
    assert main(["bench", "--orders", "4,8", "--voxels", "20000", "--repeats", "2", "--out", p]) == 0
    lines = open(p).read().strip().splitlines()
    assert lines[0] == "direction,order,voxels,method,seconds,max_dev" and len(lines) == 1 + 2 * 2 * 2
    for ln in lines[1:]:
        d, o, v, m, s, dev = ln.split(",")
        assert m in ("gpu", "gpu-e2e") and float(s) > 0 and float(dev) < 1e-4


def test_cli_lsc_with_kernel_json(tmp_path):
    """lsc --kernel with the reference-written kernel document (2 -> 3 shells, rings [5, 7], order 4 -> 2)."""
    out = str(tmp_path / "lsck.nii.gz")
    assert main(["lsc", "--sh", j("cli_sh.nii.gz"), *GR, "--kernel", j("kernel_ref.json"), "--order-out", "2",
                 "--out", out]) == 0
    assert port.rel_err(rd(out), rd(j("cli_lsc_k.nii.gz"))) <= 1e-4
