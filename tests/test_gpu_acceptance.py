"""The reference's acceptance criteria (/root/reference/pkg/tests/test_acceptance.py, SPEC criteria 1-10), run
through the sm_100a path.  The reference states float64 bounds (1e-9 ... 1e-12); the device computes in fp32,
so each bound here is the fp32 counterpart (north_star: 1e-5 for SH coefficients and signals, 1e-4 for LSC
outputs), stated per criterion.  Criterion 4 (the reference's batched-vs-naive CPU speed-up) becomes: the GPU
transform at 450k voxels, order 8, is >= 5x faster than the float64 batched host product and its speed-up
grows with the voxel count."""

import time

import numpy as np
import pytest
import torch

import paper_1808_01517_b200 as dl
from oracle import port
from paper_1808_01517_b200 import dwio, functional as F
from paper_1808_01517_b200.cli import main
from paper_1808_01517_b200.directions import unit_sphere_directions
from paper_1808_01517_b200.geometry import high_degree_energy_fraction

pytestmark = pytest.mark.gpu
TWO_SQRT_PI = 2.0 * np.sqrt(np.pi)
PI5 = np.pi / 5


@pytest.fixture(scope="module", autouse=True)
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1808_01517_b200._build import build_library

    build_library()


def band_limited(seed, n, order, nvox, scale=0.2):
    rng = np.random.default_rng(seed)
    d = unit_sphere_directions(n)
    c = rng.normal(size=(dl.coeff_count(order), nvox)) * scale
    c[0] = TWO_SQRT_PI
    sig = (dl.eval_basis(d, order) @ c).astype(np.float32)
    return d, F.DwiVolume(torch.tensor(sig.reshape(1, n, nvox, 1, 1), device="cuda")), c


def random_sh(seed, order, nvox, shells=1, scale=0.2):
    r = dl.coeff_count(order)
    c = np.random.default_rng(seed).normal(size=(1, shells * r, nvox, 1, 1)) * scale
    for s in range(shells):
        c[0, s * r] = TWO_SQRT_PI
    return F.ShVolume(torch.tensor(c, dtype=torch.float32, device="cuda"), dl.ShBasisSpec(order), shells)


def N(t):
    return t.detach().double().cpu().numpy()


def test_criterion_01_round_trip():
    """Round trip of 100 band-limited voxels (order 4, 30 dirs, lambda 0): 1e-5 normwise (fp32)."""
    d, vol, _ = band_limited(101, 30, 4, 100)
    back = F.sh_to_signal(F.signal_to_sh(vol, dl.make_fit_operator(d, 4, 0.0)), d)
    assert port.rel_err(N(back.data), N(vol.data)) <= 1e-5


def test_criterion_02_constant_signal():
    """A constant signal fits to c0 = 2 sqrt(pi), all other coefficients 0, for lambda in {0, .006, .06}."""
    d = unit_sphere_directions(30)
    vol = F.DwiVolume(torch.ones((1, 30, 5, 1, 1), device="cuda"))
    for lam in (0.0, 0.006, 0.06):
        c = N(F.signal_to_sh(vol, dl.make_fit_operator(d, 4, lam)).data)[0, :, 0, 0, 0]
        assert abs(c[0] - TWO_SQRT_PI) <= 1e-5 * TWO_SQRT_PI and np.max(np.abs(c[1:])) <= 1e-5


def test_criterion_03_oracle_equivalence():
    """The device fit equals the float64 per-voxel solver (oracle) on 10k voxels, orders 2-8, 90 dirs: 1e-5."""
    for order in (2, 4, 6, 8):
        d, vol, _ = band_limited(300 + order, 90, order, 10_000)
        got = N(F.signal_to_sh(vol, dl.make_fit_operator(d, order, 0.006)).data)
        M, _, _ = port.fit_operator(d, order, 0.006)
        ref = port.signal_to_sh(N(vol.data), M, 1)
        assert port.rel_err(got, ref) <= 1e-5, order


def test_criterion_04_performance_shape():
    """450k voxels, order 8, 90 dirs: the device transform is >= 5x the float64 batched host product (BLAS on
    one thread, as the reference's bench pins it), and device throughput does not fall as the voxel count grows
    (15% allowance per step, the reference criterion's measurement allowance)."""
    from threadpoolctl import threadpool_limits

    d = unit_sphere_directions(90)
    op = dl.make_fit_operator(d, 8, 0.006)
    rates = []
    for nvox in (1_000, 10_000, 100_000, 450_000):
        x = np.random.default_rng(nvox).uniform(0.1, 1.2, size=(90, nvox))
        vol = F.DwiVolume(torch.tensor(x.reshape(1, 90, nvox, 1, 1), dtype=torch.float32, device="cuda"),
                          check_finite=False)
        F.signal_to_sh(vol, op)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            F.signal_to_sh(vol, op)
        e1.record()
        torch.cuda.synchronize()
        dev_s = e0.elapsed_time(e1) / 20 / 1e3
        rates.append(nvox / dev_s)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        for _ in range(3):
            op.fit_matrix @ x
        host_s = (time.perf_counter() - t0) / 3
    assert host_s / dev_s >= 5.0, (host_s, dev_s)
    assert all(b >= 0.85 * a for a, b in zip(rates, rates[1:])), rates
    assert rates[-1] > rates[0], rates


def test_criterion_05_lsc_identity():
    """Identity kernel at lambda 0 reproduces the coefficients: 1e-4 (LSC, fp32)."""
    d = unit_sphere_directions(30)
    geom = dl.build_lsc_geometry(d, [5], PI5, 4, 4, 0.0)
    sh = random_sh(505, 4, 100)
    out = F.lsc_forward(sh, dl.make_identity_kernel([5]), geom)
    assert port.rel_err(N(out.data), N(sh.data)) <= 1e-4


def test_criterion_06_lsc_smoothing():
    """Moving average (5, pi/5) lowers the mean l >= 2 energy fraction and keeps a constant (1e-5)."""
    d = unit_sphere_directions(30)
    geom = dl.build_lsc_geometry(d, [5], PI5, 4, 4, 0.0)
    k = dl.make_moving_average_kernel([5])
    sh = random_sh(606, 4, 100)
    out = F.lsc_forward(sh, k, geom)
    fi = high_degree_energy_fraction(N(sh.data)[0].reshape(15, -1), 4)
    fo = high_degree_energy_fraction(N(out.data)[0].reshape(15, -1), 4)
    assert np.mean(fo / fi) < 1.0 and np.mean(fo) < np.mean(fi)
    const = np.zeros((1, 15, 10, 1, 1))
    const[0, 0] = TWO_SQRT_PI
    cs = F.ShVolume(torch.tensor(const, dtype=torch.float32, device="cuda"), dl.ShBasisSpec(4))
    assert port.rel_err(N(F.lsc_forward(cs, k, geom).data), const) <= 1e-5


def test_criterion_07_multi_shell():
    """Zero cross-shell weights reduce a 2-shell LSC to two single-shell LSCs (1e-5 of the output)."""
    d = unit_sphere_directions(30)
    geom = dl.build_lsc_geometry(d, [5], PI5, 4, 4, 0.0)
    rng = np.random.default_rng(707)
    wa, wb = rng.normal(size=6), rng.normal(size=6)
    w = np.zeros((2, 2, 6))
    w[0, 0], w[1, 1] = wa, wb
    b = rng.normal(size=2)
    sh2 = random_sh(708, 4, 50, shells=2)
    out2 = N(F.lsc_forward(sh2, dl.LscKernel(w, b), geom).data)
    for s, ws, bs in ((0, wa, b[0]), (1, wb, b[1])):
        single = F.ShVolume(sh2.data[:, s * 15:(s + 1) * 15].contiguous(), dl.ShBasisSpec(4))
        out1 = N(F.lsc_forward(single, dl.LscKernel(ws.reshape(1, 1, 6), np.array([bs])), geom).data)
        assert port.rel_err(out2[:, s * 15:(s + 1) * 15], out1) <= 1e-5


def test_criterion_08_regularization_path():
    """Along lambda = 0, 1e-3, 1e-2, 1e-1 the device fit's residual does not fall and its Laplace-Beltrami
    penalty does not rise (fp32 slack 1e-5 relative)."""
    d = unit_sphere_directions(30)
    B = dl.eval_basis(d, 4)
    pen = dl.laplace_beltrami_diag(4)
    sig = np.random.default_rng(808).normal(size=(30, 20)) + 1.0
    vol = F.DwiVolume(torch.tensor(sig.reshape(1, 30, 20, 1, 1), dtype=torch.float32, device="cuda"))
    res, pens = [], []
    for lam in (0.0, 1e-3, 1e-2, 1e-1):
        c = N(F.signal_to_sh(vol, dl.make_fit_operator(d, 4, lam)).data)[0, :, :, 0, 0]
        res.append(np.linalg.norm(B @ c - sig, axis=0))
        pens.append(np.sum(pen[:, None] * c * c, axis=0))
    for a, b in zip(res, res[1:]):
        assert np.all(b >= a * (1 - 1e-5) - 1e-6)
    for a, b in zip(pens, pens[1:]):
        assert np.all(b <= a * (1 + 1e-5) + 1e-6)


def test_criterion_09_io_and_malformed_tables(tmp_path):
    """NIfTI float32 round trip; the CLI rejects every malformed gradient table with exit 2 and no output."""
    vol = np.random.default_rng(909).normal(size=(8, 8, 8, 20))
    p = str(tmp_path / "vol.nii.gz")
    dwio.write_nifti(p, vol)
    data, _, _ = dwio.read_nifti(p)
    assert np.max(np.abs(data - vol) / np.maximum(np.abs(vol), 1e-12)) <= 1e-6
    dwi = str(tmp_path / "dwi.nii.gz")
    dwio.write_nifti(dwi, np.ones((2, 2, 2, 3)))
    good_vecs = "0 1 0\n0 0 1\n0 0 0\n"
    bad = {"four-row bvecs": ("0 1000 1000\n", good_vecs + "1 1 1\n"), "count mismatch": ("0 1000\n", good_vecs),
           "non-numeric bval": ("0 10oo 1000\n", good_vecs), "non-numeric bvec": ("0 1000 1000\n", "0 x 0\n0 0 1\n0 0 0\n"),
           "non-finite bval": ("0 nan 1000\n", good_vecs), "non-finite bvec": ("0 1000 1000\n", "0 inf 0\n0 0 1\n0 0 0\n"),
           "zero dwi vector": ("0 1000 1000\n", "0 1 0\n0 0 0\n0 0 0\n"), "ragged bvecs": ("0 1000 1000\n", "0 1 0\n0 0\n0 0 0\n"),
           "empty bvals": ("\n", good_vecs)}
    out = tmp_path / "never.nii.gz"
    for name, (bv, bvec) in bad.items():
        (tmp_path / "b.bval").write_text(bv)
        (tmp_path / "b.bvec").write_text(bvec)
        code = main(["signal2sh", "--dwi", dwi, "--bvals", str(tmp_path / "b.bval"), "--bvecs",
                     str(tmp_path / "b.bvec"), "--out", str(out)])
        assert code == 2, name
        assert not out.exists(), name


def test_criterion_10_end_to_end_cli(tmp_path):
    """Files only: a band-limited acquisition (1 b0 + 30 dirs, written here; the phantom command is out of
    scope) -> signal2sh -> lsc (moving average) -> sh2signal; smoothing lowers the l >= 2 energy fraction."""
    d = unit_sphere_directions(30)
    rng = np.random.default_rng(10)
    c = port.bandlimited_coeffs(rng, 4, 100)
    sig = (dl.eval_basis(d, 4) @ c).T.reshape(5, 5, 4, 30)
    acq = np.concatenate([np.ones((5, 5, 4, 1)), sig], axis=3) * 1000.0
    pre = str(tmp_path / "ph")
    dwio.write_nifti(pre + ".nii.gz", acq)
    dwio.write_bvals_bvecs(np.r_[0.0, [1000.0] * 30], np.vstack([np.zeros(3), d]), pre + ".bvals", pre + ".bvecs")
    g = ["--bvals", pre + ".bvals", "--bvecs", pre + ".bvecs"]
    sh, sm, out = (str(tmp_path / n) for n in ("sh.nii.gz", "smooth.nii.gz", "signal.nii.gz"))
    assert main(["signal2sh", "--dwi", pre + ".nii.gz", *g, "--order", "4", "--lambda", "0", "--out", sh]) == 0
    assert main(["lsc", "--sh", sh, *g, "--shell", "1000", "--moving-average", f"5,{PI5}", "--lambda", "0",
                 "--out", sm]) == 0
    assert main(["sh2signal", "--sh", sm, *g, "--shell", "1000", "--order", "4", "--out", out]) == 0
    before, after = dwio.read_nifti(sh)[0], dwio.read_nifti(sm)[0]
    fb = high_degree_energy_fraction(before.reshape(-1, 15).T, 4)
    fa = high_degree_energy_fraction(after.reshape(-1, 15).T, 4)
    assert np.mean(fa / fb) < 1.0 and np.mean(fa) < np.mean(fb)
    y = dwio.read_nifti(out)[0]
    assert y.shape == (5, 5, 4, 30) and np.isfinite(y).all()
