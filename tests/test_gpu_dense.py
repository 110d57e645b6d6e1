"""The small float64 kernels of the stacked-LSC path (csrc/dense.cu) against torch float64 on the same device."""

import numpy as np
import pytest
import torch

from paper_1808_01517_b200 import _lib, ops

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1808_01517_b200._build import build_library

    build_library()
    return torch.device("cuda:0")


@pytest.mark.parametrize("m,n,k,ta,tb", [(135, 135, 135, False, False), (90, 1, 135, False, False),
                                          (135, 135, 135, True, False), (45, 17, 33, False, True),
                                          (1, 1, 1, True, True), (200, 3, 1, False, False)])
def test_gemm_f64(dev, m, n, k, ta, tb):
    g = torch.Generator(device=dev).manual_seed(m * 7 + n * 3 + k)
    A = torch.randn((k, m) if ta else (m, k), dtype=torch.float64, device=dev, generator=g)
    B = torch.randn((n, k) if tb else (k, n), dtype=torch.float64, device=dev, generator=g)
    C0 = torch.randn((m, n), dtype=torch.float64, device=dev, generator=g)
    ref = (A.T if ta else A) @ (B.T if tb else B)
    got = ops.gemm_f64(A, B, ta=ta, tb=tb)
    assert torch.allclose(got, ref, rtol=1e-12, atol=1e-12)
    got2 = ops.gemm_f64(A, B, ta=ta, tb=tb, C=C0.clone(), alpha=-0.5, beta=2.0)
    assert torch.allclose(got2, -0.5 * ref + 2.0 * C0, rtol=1e-12, atol=1e-12)


def test_lsc_dw_from_dl(dev):
    rng = np.random.default_rng(3)
    so, si, K, ro, ri = 3, 2, 6, 45, 28
    fold = torch.tensor(rng.normal(size=(K, ro, ri)), dtype=torch.float32, device=dev)
    dL = torch.tensor(rng.normal(size=(so * ro, si * ri)), dtype=torch.float64, device=dev)
    dW = torch.empty((so, si, K), dtype=torch.float32, device=dev)
    _lib.call("dl_lsc_dw_from_dl_f64", ops._p(dL), ops._p(fold), ops._p(dW), so, si, K, ro, ri, ops._stream())
    ref = torch.einsum("krt,orst->osk", fold.double(), dL.view(so, ro, si, ri))
    assert torch.allclose(dW.double(), ref, rtol=1e-6, atol=1e-9)
