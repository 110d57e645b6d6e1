"""Host I/O of the ingest path (dwio.py) against the reference's files and its own test cases
(/root/reference/pkg/tests/test_dwio.py), plus the volume-selection checks of normalize_b0 (CPU only)."""

import gzip
import os
import struct

import numpy as np
import pytest

from conftest import ROOT
from paper_1808_01517_b200 import dwio
from paper_1808_01517_b200.errors import (GradientParseError, MissingB0Error, NiftiDatatypeError, NiftiMagicError,
                                          NiftiTruncatedError, ShapeError)
from paper_1808_01517_b200.ingest import select_volumes

G = os.path.join(ROOT, "tests", "golden", "ingest")


@pytest.fixture(scope="module")
def exp():
    return np.load(os.path.join(G, "expected.npz"))


def test_read_reference_written_file(exp):
    data, affine, hdr = dwio.read_nifti(os.path.join(G, "acq.nii.gz"))
    assert np.array_equal(data, exp["data"])          # int16 * 0.5 + 10, exact in float64
    assert np.allclose(affine, exp["affine"])
    raw = dwio.read_nifti_raw(os.path.join(G, "acq.nii.gz"))
    assert raw.dtype_code == 4 and raw.data.dtype == np.int16 and raw.shape == exp["data"].shape
    assert raw.scaled and raw.slope == 0.5 and raw.inter == 10.0
    X, Y, Z, V = raw.shape
    assert raw.strides() == (1, X, X * Y, X * Y * Z)


def test_gradient_table_and_selection(exp):
    s = dwio.read_bvals_bvecs(os.path.join(G, "acq.bval"), os.path.join(G, "acq.bvec"))
    assert list(s.b0_indices) == [0, 4] and s.shell_bvalues() == [1000.0, 2000.0]
    assert np.allclose(np.linalg.norm(s.directions[s.shells[0].indices], axis=1), 1.0)
    b0, table = select_volumes(s, s.n)
    sel = np.concatenate([t.indices for t in table])
    assert np.array_equal(s.bvals[sel], exp["sub_bvals"])
    assert np.allclose(s.directions[sel], exp["sub_dirs"])


@pytest.mark.parametrize("bvals,b0,groups", [
    ([0, 1000, 1000, 2000], [0], [(1000, [1, 2]), (2000, [3])]),
    ([5, 990, 1010, 1040, 3000], [0], [(1015, [1, 2, 3]), (3000, [4])]),      # within tolerance merge, round to 5
    ([0, 1000, 1100], [0], [(1000, [1]), (1100, [2])]),                     # gap beyond tolerance splits
    ([40, 60], [0], [(60, [1])]),                                           # near-zero goes to b0
])
def test_detect_shells(bvals, b0, groups):
    got_b0, shells = dwio.detect_shells(bvals)
    assert list(got_b0) == b0
    assert [(s.bvalue, list(s.indices)) for s in shells] == [(float(b), i) for b, i in groups]


def test_detect_shells_bad_tolerance():
    with pytest.raises(ValueError):
        dwio.detect_shells([0, 1000], tolerance=0)


def test_selection_errors():
    with pytest.raises(MissingB0Error):
        select_volumes([1000.0, 1000.0], 2)
    with pytest.raises(ShapeError, match="unequal"):
        select_volumes([0.0, 1000.0, 1000.0, 2000.0], 4)
    _, t = select_volumes([0.0, 1000.0, 1000.0, 2000.0], 4, shells=[2000.0])
    assert len(t) == 1 and list(t[0].indices) == [3]
    with pytest.raises(ShapeError, match="describes"):
        select_volumes([0.0, 1000.0], 3)
    with pytest.raises(ValueError, match="no shell near"):
        select_volumes([0.0, 1000.0], 2, shells=[3000.0])


def test_bvec_layouts_and_errors(tmp_path):
    b, v = tmp_path / "b", tmp_path / "v"
    b.write_text("0 1000 1000 2000\n")
    v.write_text("0 0 0\n1 0 0\n0 2 0\n0 0 3\n")         # N x 3 layout
    s = dwio.read_bvals_bvecs(str(b), str(v))
    assert s.n == 4 and np.allclose(s.directions[2], [0, 1, 0])
    v.write_text("0 1 0 0\n0 0 1 0\n0 0 0 1\n")            # 3 x N layout
    assert np.allclose(dwio.read_bvals_bvecs(str(b), str(v)).directions[3], [0, 0, 1])
    b.write_text("0 1000 1000\n")
    v.write_text("0 1 0 0\n0 0 1 0\n")
    with pytest.raises(GradientParseError):
        dwio.read_bvals_bvecs(str(b), str(v))
    v.write_text("0 1 0\n0 0 0\n0 0 0\n")
    with pytest.raises(GradientParseError, match="zero direction"):
        dwio.read_bvals_bvecs(str(b), str(v))
    v.write_text("0 1 x\n0 0 1\n0 0 0\n")
    with pytest.raises(GradientParseError, match="non-numeric"):
        dwio.read_bvals_bvecs(str(b), str(v))


@pytest.mark.parametrize("dtype", [np.uint8, np.int16, np.int32, np.float32, np.float64])
@pytest.mark.parametrize("suffix", [".nii", ".nii.gz"])
def test_write_read_round_trip(tmp_path, dtype, suffix):
    rng = np.random.default_rng(3)
    a = (rng.uniform(0, 100, size=(4, 3, 5, 2))).astype(dtype)
    aff = np.array([[0, -2.0, 0, 5], [1.5, 0, 0, -3], [0, 0, 2.5, 1], [0, 0, 0, 1]])
    p = str(tmp_path / ("v" + suffix))
    dwio.write_nifti(p, a, affine=aff, dtype=dtype)
    d, got_aff, _ = dwio.read_nifti(p)
    assert np.array_equal(d, a.astype(np.float64)) and np.allclose(got_aff, aff)


def _header(p):
    with open(p, "rb") as fh:
        return bytearray(fh.read())


def test_nifti_errors(tmp_path):
    p = str(tmp_path / "v.nii")
    dwio.write_nifti(p, np.ones((2, 2, 2), np.float32))
    good = _header(p)
    cases = {
        "magic": (lambda h: struct.pack_into("<4s", h, 344, b"ni1\x00"), NiftiMagicError),
        "dtype": (lambda h: struct.pack_into("<h", h, 70, 32), NiftiDatatypeError),
        "negdim": (lambda h: struct.pack_into("<h", h, 42, -2), NiftiMagicError),
        "offset": (lambda h: struct.pack_into("<f", h, 108, 10.0), NiftiMagicError),
        "size": (lambda h: struct.pack_into("<i", h, 0, 1234), NiftiMagicError),
    }
    for name, (patch, exc) in cases.items():
        h = bytearray(good)
        patch(h)
        q = str(tmp_path / f"{name}.nii")
        open(q, "wb").write(bytes(h))
        with pytest.raises(exc):
            dwio.read_nifti(q)
    q = str(tmp_path / "short.nii")
    open(q, "wb").write(bytes(good[:200]))
    with pytest.raises(NiftiTruncatedError):
        dwio.read_nifti(q)
    open(q, "wb").write(bytes(good[:-8]))
    with pytest.raises(NiftiTruncatedError):
        dwio.read_nifti(q)


def test_byte_swapped_file(tmp_path):
    a = np.arange(24, dtype=np.int16).reshape(2, 3, 4)
    p = str(tmp_path / "le.nii")
    dwio.write_nifti(p, a, dtype=np.int16)
    h = _header(p)
    be = bytearray(h)
    # re-encode the fields the reader uses as big-endian
    for off, fmt in [(0, "i"), (40, "8h"), (70, "hh"), (76, "8f"), (108, "fff"), (252, "hh"), (280, "4f"),
                     (296, "4f"), (312, "4f")]:
        struct.pack_into(">" + fmt, be, off, *struct.unpack_from("<" + fmt, h, off))
    be[352:] = a.astype(">i2").tobytes(order="F")
    q = str(tmp_path / "be.nii")
    open(q, "wb").write(bytes(be))
    d, _, _ = dwio.read_nifti(q)
    assert np.array_equal(d, a)
    r = dwio.read_nifti_raw(q)
    assert r.data.dtype.isnative and np.array_equal(r.data.reshape(r.shape, order="F"), a)


def test_gzip_matches_plain(tmp_path):
    a = np.random.default_rng(1).normal(size=(3, 4, 5)).astype(np.float32)
    dwio.write_nifti(str(tmp_path / "a.nii"), a)
    dwio.write_nifti(str(tmp_path / "a.nii.gz"), a)
    with gzip.open(str(tmp_path / "a.nii.gz")) as fh:
        assert fh.read() == open(str(tmp_path / "a.nii"), "rb").read()


# --------------------------------------------------------------------------- kernel interchange (lsc.py:223-277)
def test_kernel_json_from_reference(tmp_path):
    from paper_1808_01517_b200 import kernel_io

    k, sizes, alpha = kernel_io.load_kernel_json(os.path.join(G, "kernel_ref.json"))
    assert sizes == (5, 7) and alpha == np.pi / 8 and k.weights.shape == (3, 2, 13)
    p = str(tmp_path / "k.json")
    kernel_io.save_kernel_json(p, k, sizes, alpha)
    import json
    ref = json.load(open(os.path.join(G, "kernel_ref.json")))
    mine = json.load(open(p))
    assert mine == ref                          # same document, value for value


def test_kernel_json_errors(tmp_path):
    import json

    from paper_1808_01517_b200 import kernel_io
    from paper_1808_01517_b200.errors import KernelMismatchError
    from paper_1808_01517_b200.geometry import LscKernel

    k = LscKernel(np.zeros((1, 1, 6)), np.zeros(1))
    with pytest.raises(KernelMismatchError):
        kernel_io.save_kernel_json(str(tmp_path / "a.json"), k, [7], 0.3)
    good = dict(shells_in=1, shells_out=1, kernel_sizes=[5], angular_distance=0.3, weights=[[[0.0] * 6]], bias=[0.0])
    for name, doc in {"missing": {k_: v for k_, v in good.items() if k_ != "bias"},
                      "shells": {**good, "shells_in": 2},
                      "length": {**good, "kernel_sizes": [6]}}.items():
        q = tmp_path / f"{name}.json"
        q.write_text(json.dumps(doc))
        with pytest.raises(KernelMismatchError):
            kernel_io.load_kernel_json(str(q))
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(KernelMismatchError):
        kernel_io.load_kernel_json(str(tmp_path / "bad.json"))


def test_module_round_trip_and_state_dict(tmp_path):
    import torch

    import paper_1808_01517_b200 as dl
    from paper_1808_01517_b200 import kernel_io
    from paper_1808_01517_b200.directions import unit_sphere_directions
    from paper_1808_01517_b200.errors import KernelMismatchError

    d = unit_sphere_directions(30)
    a = dl.LocalSphericalConvolution(2, 3, 4, 4, d, [5, 7], angular_distance=np.pi / 8)
    b = dl.LocalSphericalConvolution(2, 3, 4, 4, d, [5, 7], angular_distance=np.pi / 8)
    kernel_io.load_module(os.path.join(G, "kernel_ref.json"), a)
    p = str(tmp_path / "m.json")
    kernel_io.save_module(p, a)
    kernel_io.load_module(p, b)
    assert torch.equal(a.sconv.weight, b.sconv.weight) and torch.equal(a.sconv.bias, b.sconv.bias)
    c = dl.LocalSphericalConvolution(2, 3, 4, 4, d, [5, 7], angular_distance=np.pi / 8)
    c.load_state_dict(a.state_dict())
    assert torch.equal(c.sconv.weight, a.sconv.weight)
    wrong = dl.LocalSphericalConvolution(2, 3, 4, 4, d, [5, 7], angular_distance=np.pi / 9)
    with pytest.raises(KernelMismatchError):
        kernel_io.load_module(p, wrong)
