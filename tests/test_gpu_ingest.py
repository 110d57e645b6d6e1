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


def _chain_for(dev, tables, order=4, seed=3):
    from paper_1808_01517_b200.directions import unit_sphere_directions  # noqa: F401

    rng = np.random.default_rng(seed)
    s = tables.shape[0]
    s2sh = dl.Signal2SH(order, tables, lb_lambda=0.006).to(dev)
    lsc = dl.LocalSphericalConvolution(s, s, order, order, tables[0], [5], lb_lambda=0.006,
                                       angular_distance=np.pi / 5).to(dev)
    lsc.load_kernel(dl.LscKernel(rng.normal(size=(s, s, 6)) / (6 * s), rng.normal(size=s) * 0.1))
    return dl.SphericalChain(s2sh, lsc, dl.SH2Signal(order, tables[0]).to(dev)), s2sh, lsc


def test_chain_from_raw_matches_reference(dev, exp):
    """normalize_b0 fused into the chain kernel == the reference's normalize_b0 output
    (expected.npz, made by sphdwi) pushed through the oracle chain, at the LSC tolerance; mask identical."""
    from oracle import port

    raw = dwio.read_nifti_raw(os.path.join(G, "acq.nii.gz"))
    scheme = dwio.read_bvals_bvecs(os.path.join(G, "acq.bval"), os.path.join(G, "acq.bvec"))
    sub = dl.normalize_b0(raw, scheme, device=dev)[0].scheme
    tables = np.stack([sub.shell_directions(b) for b in sub.shell_bvalues()])
    chain, s2sh, lsc = _chain_for(dev, tables)
    y, mask, sub2 = dl.chain_from_raw(chain, raw, scheme, device=dev)
    assert tuple(y.shape) == (1, 2 * 6, 9, 7, 6) and not y.is_contiguous()   # stored (x-fastest) voxel order
    assert np.array_equal(mask.cpu().numpy(), exp["mask"]) and np.array_equal(sub2.bvals, exp["sub_bvals"])
    Ms = [op.fit_matrix for op in s2sh.operators]
    geo = port.lsc_geometry(tables[0], [5], np.pi / 5, 4, 4, 0.006)
    w = lsc.sconv.weight.detach().double().cpu().numpy()[:, :, 0, :]
    b = lsc.sconv.bias.detach().double().cpu().numpy()
    y_ref = port.chain_forward(exp["vol"], Ms, geo, w, b, port.eval_basis(tables[0], 4), 2)
    assert port.rel_err(y.double().cpu().numpy(), y_ref) <= 1e-4
    # and equal to the two-pass path (normalize_b0 volume -> fused chain) at the same tolerance
    vol, _ = dl.normalize_b0(raw, scheme, device=dev)
    with torch.no_grad():
        y2 = chain(vol.data)
    assert port.rel_err(y.double().cpu().numpy(), y2.double().cpu().numpy()) <= 1e-5


@pytest.mark.parametrize("kind", ["f32_fortran", "i16_fortran_scaled", "c_order_fallback"])
def test_chain_from_raw_layouts(dev, kind):
    """Larger volumes (several 128-voxel tiles + a tail): float32 and scaled int16 stored x-fastest run fused; a
    C-ordered in-memory array takes the two-pass fallback; all match normalize_b0 -> chain."""
    from oracle import port

    rng = np.random.default_rng(11)
    X, Y, Z = 38, 21, 13                       # nvox = 10374 (even): 81 tiles + a tail of 6
    bvals = np.array([0.0] + [1000.0] * 30 + [0.0] + [2000.0] * 30)
    dirs = rng.normal(size=(bvals.size, 3))
    scheme_dirs = dirs / np.linalg.norm(dirs, axis=1, keepdims=True)
    scheme = dwio.GradientScheme(scheme_dirs, bvals, np.array([0, 31]),
                                 (dwio.Shell(1000.0, np.arange(1, 31)), dwio.Shell(2000.0, np.arange(32, 62))),
                                 dwio.B0_THRESHOLD)
    stored = rng.uniform(200.0, 3000.0, size=(X, Y, Z, bvals.size))
    stored[..., [0, 31]] += 2000.0
    if kind == "i16_fortran_scaled":
        arr = stored.astype(np.int16)
        raw = dwio.NiftiRaw(np.asfortranarray(arr).ravel(order="F"), arr.shape, dwio.CODE_OF[np.dtype(np.int16)],
                            0.5, 10.0, np.eye(4), {})
        ref_in = arr.astype(np.float64) * 0.5 + 10.0
    elif kind == "f32_fortran":
        arr = stored.astype(np.float32)
        raw = torch.from_numpy(np.asfortranarray(arr))
        ref_in = arr.astype(np.float64)
    else:
        arr = stored.astype(np.float32)
        raw = np.ascontiguousarray(arr)
        ref_in = arr.astype(np.float64)
    tables = np.stack([scheme_dirs[1:31], scheme_dirs[32:62]])
    chain, s2sh, lsc = _chain_for(dev, tables)
    y, mask, _ = dl.chain_from_raw(chain, raw, scheme, device=dev)
    assert y.is_contiguous() == (kind == "c_order_fallback")
    b0 = ref_in[..., [0, 31]].mean(axis=3)
    xn = np.moveaxis(ref_in[..., list(range(1, 31)) + list(range(32, 62))] / b0[..., None], 3, 0)[None]
    Ms = [op.fit_matrix for op in s2sh.operators]
    geo = port.lsc_geometry(tables[0], [5], np.pi / 5, 4, 4, 0.006)
    w = lsc.sconv.weight.detach().double().cpu().numpy()[:, :, 0, :]
    b = lsc.sconv.bias.detach().double().cpu().numpy()
    y_ref = port.chain_forward(xn, Ms, geo, w, b, port.eval_basis(tables[0], 4), 2)
    assert port.rel_err(y.double().cpu().numpy(), y_ref) <= 1e-4
    assert not mask.any()


@pytest.mark.parametrize("case", ["stacked_two_layers", "odd_nvox_fallback"])
def test_chain_from_raw_more(dev, case):
    """Stacked LSC layers through the raw-input kernel (folded operator), and an odd voxel count (the two-pass
    fallback): both equal normalize_b0 -> chain."""
    rng = np.random.default_rng(21)
    X, Y, Z = (10, 9, 7) if case == "stacked_two_layers" else (9, 7, 5)      # 630 (even) / 315 (odd)
    bvals = np.array([0.0] + [1000.0] * 30 + [0.0] + [2000.0] * 30)
    dirs = rng.normal(size=(bvals.size, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    scheme = dwio.GradientScheme(dirs, bvals, np.array([0, 31]),
                                 (dwio.Shell(1000.0, np.arange(1, 31)), dwio.Shell(2000.0, np.arange(32, 62))),
                                 dwio.B0_THRESHOLD)
    arr = (rng.uniform(200.0, 3000.0, size=(X, Y, Z, bvals.size)) + 1000.0 * np.isin(np.arange(bvals.size), [0, 31])
           ).astype(np.int16)
    raw = dwio.NiftiRaw(np.asfortranarray(arr).ravel(order="F"), arr.shape, dwio.CODE_OF[np.dtype(np.int16)],
                        0.0, 0.0, np.eye(4), {})
    tables = np.stack([dirs[1:31], dirs[32:62]])
    s2sh = dl.Signal2SH(4, tables, lb_lambda=0.006).to(dev)
    layers = []
    for k in range(2 if case == "stacked_two_layers" else 1):
        m = dl.LocalSphericalConvolution(2, 2, 4, 4, tables[0], [5], lb_lambda=0.006, angular_distance=np.pi / 5).to(dev)
        m.load_kernel(dl.LscKernel(rng.normal(size=(2, 2, 6)) / 12, rng.normal(size=2) * 0.1))
        layers.append(m)
    chain = dl.SphericalChain(s2sh, layers if len(layers) > 1 else layers[0], dl.SH2Signal(4, tables[0]).to(dev))
    y, _, _ = dl.chain_from_raw(chain, raw, scheme, device=dev)
    assert y.is_contiguous() == (case == "odd_nvox_fallback")
    vol, _ = dl.normalize_b0(raw, scheme, device=dev)
    with torch.no_grad():
        y2 = chain(vol.data)
    from oracle import port

    assert port.rel_err(y.double().cpu().numpy(), y2.double().cpu().numpy()) <= 1e-5
