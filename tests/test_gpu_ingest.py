"""Ingest kernel (dl_normalize_b0_f32, csrc/ingest.cu) against the reference's normalize_b0 outputs
(tests/golden/ingest/, made by tests/golden/make_ingest_golden.py with the real sphdwi).

Tolerance: the kernel works in float64 and rounds once to fp32, so it must agree with the reference's float64
result to fp32 rounding: max |got - ref| <= 2^-24 * |ref| elementwise; the exclusion mask must be identical.
"""

import os

import numpy as np
import pytest
import torch

import paper_1808_01517_b200 as dl
from conftest import ROOT
from paper_1808_01517_b200 import dwio

pytestmark = pytest.mark.gpu
G = os.path.join(ROOT, "tests", "golden", "ingest")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1808_01517_b200._build import build_library

    build_library()
    return torch.device("cuda:0")


@pytest.fixture(scope="module")
def exp():
    return np.load(os.path.join(G, "expected.npz"))


def close_fp32(got, ref):
    got = got.detach().double().cpu().numpy()
    assert got.shape == ref.shape
    assert np.all(np.abs(got - ref) <= 2.0 ** -24 * np.abs(ref) + 1e-300), np.max(np.abs(got - ref))


def test_load_dwi_matches_reference(dev, exp):
    vol, mask, scheme = dl.load_dwi(os.path.join(G, "acq.nii.gz"), os.path.join(G, "acq.bval"),
                                    os.path.join(G, "acq.bvec"), device=dev)
    close_fp32(vol.data, exp["vol"])
    assert np.array_equal(mask.cpu().numpy(), exp["mask"])
    assert vol.shells == 2 and np.array_equal(scheme.bvals, exp["sub_bvals"])
    vol2, mask2, _ = dl.load_dwi(os.path.join(G, "acq.nii.gz"), os.path.join(G, "acq.bval"),
                                 os.path.join(G, "acq.bvec"), shells=[2000.0], device=dev)
    close_fp32(vol2.data, exp["vol_b2000"])
    assert np.array_equal(mask2.cpu().numpy(), exp["mask_b2000"])


@pytest.mark.parametrize("kind", ["numpy64", "torch64", "torch32_fortran"])
def test_in_memory_layouts(dev, exp, kind):
    mem = exp["mem"]
    bvals = [0.0, 0.0, 1000.0, 1000.0, 1000.0, 2000.0, 2000.0]
    if kind == "numpy64":
        raw = mem
    elif kind == "torch64":
        raw = torch.tensor(mem, device=dev)
    else:   # x-fastest fp32 tensor (the NIfTI order): the kernel's x-tiled path, checked on the fp32 input
        raw = torch.from_numpy(np.asfortranarray(mem.astype(np.float32)))
        assert raw.stride()[0] == 1
    vol, mask = dl.normalize_b0(raw, bvals, shells=[1000.0], device=dev)
    if kind == "torch32_fortran":
        ref64 = mem.astype(np.float32).astype(np.float64)
        b0 = ref64[..., :2].mean(axis=3)
        with np.errstate(divide="ignore", invalid="ignore"):
            ref = np.where(b0[None, ..., None] <= 1e-6 * b0.max(), 0.0, ref64[None, ..., 2:5] / b0[None, ..., None])
        close_fp32(vol.data, np.moveaxis(ref, 4, 1))
    else:
        close_fp32(vol.data, exp["vol_mem"])
    assert np.array_equal(mask.cpu().numpy(), exp["mask_mem"])


def test_integer_types_and_scaling(dev):
    rng = np.random.default_rng(5)
    X, Y, Z, V = 37, 5, 33, 6            # tiles with tails in x and z
    bvals = [0.0, 1000.0, 1000.0, 0.0, 1000.0, 1000.0]
    for dtype in (np.uint8, np.int16, np.int32):
        stored = rng.integers(1, 120, size=(X, Y, Z, V)).astype(dtype)
        raw = dwio.NiftiRaw(np.asfortranarray(stored).ravel(order="F"), stored.shape, dwio.CODE_OF[np.dtype(dtype)],
                            0.25, 3.0, np.eye(4), {})
        vol, mask = dl.normalize_b0(raw, bvals, device=dev)
        f = stored.astype(np.float64) * 0.25 + 3.0
        b0 = (f[..., 0] + f[..., 3]) / 2.0
        ref = np.moveaxis(f[..., [1, 2, 4, 5]] / b0[..., None], 3, 0)[None]
        close_fp32(vol.data, ref)
        assert not mask.any()


def test_ingest_feeds_the_chain(dev, exp):
    vol, _, scheme = dl.load_dwi(os.path.join(G, "acq.nii.gz"), os.path.join(G, "acq.bval"),
                                 os.path.join(G, "acq.bvec"), device=dev)
    tables = np.stack([scheme.shell_directions(b) for b in scheme.shell_bvalues()])
    s2sh = dl.Signal2SH(4, tables, lb_lambda=0.006).to(dev)
    c = s2sh(vol.data)
    assert c.shape == (1, 2 * 15, 9, 7, 6) and torch.isfinite(c).all()


def test_in_memory_256x256_grid_z_chunks(dev):
    """A C-contiguous (X, Y, Z, V) array with X * Y = 65536 > 65535 (the CUDA grid.z cap): ingest_k walks the
    (x, y) plane in grid.z chunks.  Also the x-fastest path with Y * ceil(n_sel / 48) > 65535."""
    rng = np.random.default_rng(9)
    X, Y, Z = 256, 256, 4
    bvals = [0.0, 1000.0, 1000.0, 2000.0, 2000.0, 0.0]
    raw = rng.uniform(50.0, 150.0, size=(X, Y, Z, len(bvals))).astype(np.float32)
    vol, mask = dl.normalize_b0(raw, bvals, device=dev)
    f = raw.astype(np.float64)
    b0 = (f[..., 0] + f[..., 5]) / 2.0
    ref = np.moveaxis(f[..., [1, 2, 3, 4]] / b0[..., None], 3, 0)[None]
    close_fp32(vol.data, ref)
    assert not mask.any()
    # x-fastest (Fortran) layout with many y rows: grid.z = Y * ceil(n_sel / 48) = 70000 * 1
    X2, Y2, Z2 = 2, 70000, 1
    raw2 = rng.uniform(50.0, 150.0, size=(X2, Y2, Z2, len(bvals))).astype(np.float32)
    t2 = torch.from_numpy(np.asfortranarray(raw2))
    assert t2.stride()[0] == 1
    vol2, _ = dl.normalize_b0(t2, bvals, device=dev)
    f2 = raw2.astype(np.float64)
    b02 = (f2[..., 0] + f2[..., 5]) / 2.0
    close_fp32(vol2.data, np.moveaxis(f2[..., [1, 2, 3, 4]] / b02[..., None], 3, 0)[None])
