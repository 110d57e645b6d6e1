"""Probe the tcgen05 conventions the fused kernels rely on (descriptor fields, operand majors,
A-from-TMEM packing, SWIZZLE_128B K-major tiles, the M=64 TMEM row mapping) against numpy.

Builds tests/cuda/umma_probe.cu (test-only) with nvcc and runs single-CTA MMAs.
"""

import ctypes
import os
import subprocess

import numpy as np
import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu

SRC = os.path.join(ROOT, "tests", "cuda", "umma_probe.cu")


@pytest.fixture(scope="module")
def probe(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = str(tmp_path_factory.mktemp("probe") / "probe.so")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-shared",
                    "-Xcompiler", "-fPIC", "-o", out, SRC], check=True)
    lib = ctypes.CDLL(out)
    lib.umma_probe.restype = ctypes.c_int
    return lib


def bf16_bits(a):
    t = torch.tensor(np.asarray(a, np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16), t.float().numpy().astype(np.float64)


def blocked(bits):
    """Core-matrix blocked no-swizzle image of an R x C bf16 matrix (umma.cuh conventions)."""
    R, C = bits.shape
    img = np.zeros(R * C, np.uint16)
    for r in range(R):
        for c in range(C):
            img[((r // 8) * (C // 8) + c // 8) * 64 + (r % 8) * 8 + c % 8] = bits[r, c]
    return img


def sw128_k(bits):
    """SWIZZLE_128B K-major image: atoms of 8 rows x 64 K-elements, [k_atom][row_group][8 x 128 B]."""
    R, K = bits.shape
    img = np.zeros(R * K, np.uint16)
    atom = (R // 8) * 512  # elements per K-atom
    for r in range(R):
        for k in range(K):
            chunk = (k % 64) // 8
            img[(k // 64) * atom + (r // 8) * 512 + (r % 8) * 64 + ((chunk ^ (r % 8)) * 8) + k % 8] = bits[r, k]
    return img


def run(lib, mode, a_img, b_img, a_words, N, K, a_desc, b_desc, M=128):
    dev = torch.device("cuda:0")
    ta = torch.tensor(a_img.view(np.uint8) if a_img is not None else np.zeros(16, np.uint8), device=dev)
    tb = torch.tensor(b_img.view(np.uint8), device=dev)
    tw = torch.tensor((a_words if a_words is not None else np.zeros(4, np.uint32)).view(np.int32), device=dev)
    d = torch.zeros(128 * N, dtype=torch.float32, device=dev)
    a_off = torch.tensor(np.asarray(a_desc[4], np.int32), device=dev)
    b_off = torch.tensor(np.asarray(b_desc[4], np.int32), device=dev)
    P = ctypes.c_void_p
    st = lib.umma_probe(mode, P(ta.data_ptr()), ta.numel(), P(tb.data_ptr()), tb.numel(), P(tw.data_ptr()),
                        P(d.data_ptr()), N, K, ctypes.c_uint32(a_desc[0]), ctypes.c_uint32(a_desc[1]), a_desc[2],
                        a_desc[3], P(a_off.data_ptr()), ctypes.c_uint32(b_desc[0]), ctypes.c_uint32(b_desc[1]),
                        b_desc[2], b_desc[3], P(b_off.data_ptr()), M)
    assert st == 0, f"cuda error {st}"
    return d.cpu().numpy().reshape(128, N).astype(np.float64)


def test_ss_kmajor_both(probe):
    rng = np.random.default_rng(0)
    M, N, K = 128, 64, 32
    ab, a = bf16_bits(rng.normal(size=(M, K)))
    wb, w = bf16_bits(rng.normal(size=(N, K)))
    ks = K // 16
    d = run(probe, 0, blocked(ab), blocked(wb), None, N, K,
            (128, (K // 8) * 128, 0, 0, [256 * k for k in range(ks)]),
            (128, (K // 8) * 128, 0, 0, [256 * k for k in range(ks)]))
    np.testing.assert_allclose(d, a @ w.T, rtol=1e-5, atol=1e-4)


def test_ss_b_mn_major(probe):
    rng = np.random.default_rng(1)
    M, N, K = 128, 96, 48
    ab, a = bf16_bits(rng.normal(size=(M, K)))
    wb, w = bf16_bits(rng.normal(size=(K, N)))      # B = w, stored K rows x N cols
    ks = K // 16
    d = run(probe, 0, blocked(ab), blocked(wb), None, N, K,
            (128, (K // 8) * 128, 0, 0, [256 * k for k in range(ks)]),
            ((N // 8) * 128, 128, 0, 1, [2 * (N // 8) * 128 * k for k in range(ks)]))
    np.testing.assert_allclose(d, a @ w, rtol=1e-5, atol=1e-4)


def test_ts_a_from_tmem(probe):
    rng = np.random.default_rng(2)
    M, N, K = 128, 48, 64
    ab, a = bf16_bits(rng.normal(size=(M, K)))
    words = (ab[:, 0::2].astype(np.uint32) | (ab[:, 1::2].astype(np.uint32) << 16))
    wb, w = bf16_bits(rng.normal(size=(N, K)))
    ks = K // 16
    d = run(probe, 1, None, blocked(wb), np.ascontiguousarray(words), N, K, (0, 0, 0, 0, [0] * ks),
            (128, (K // 8) * 128, 0, 0, [256 * k for k in range(ks)]))
    np.testing.assert_allclose(d, a @ w.T, rtol=1e-5, atol=1e-4)


def test_ts_a_from_tmem_b_mn_major(probe):
    rng = np.random.default_rng(3)
    M, N, K = 128, 96, 48
    ab, a = bf16_bits(rng.normal(size=(M, K)))
    words = (ab[:, 0::2].astype(np.uint32) | (ab[:, 1::2].astype(np.uint32) << 16))
    wb, w = bf16_bits(rng.normal(size=(K, N)))
    ks = K // 16
    d = run(probe, 1, None, blocked(wb), np.ascontiguousarray(words), N, K, (0, 0, 0, 0, [0] * ks),
            ((N // 8) * 128, 128, 0, 1, [2 * (N // 8) * 128 * k for k in range(ks)]))
    np.testing.assert_allclose(d, a @ w, rtol=1e-5, atol=1e-4)


def test_ss_sw128_kmajor_gram(probe):
    rng = np.random.default_rng(4)
    M, N, K = 128, 144, 128
    gb, g = bf16_bits(rng.normal(size=(M, K)))     # g channels x voxels
    cb, c = bf16_bits(rng.normal(size=(N, K)))     # c channels x voxels
    offs_a = [(k // 4) * (M // 8) * 1024 + (k % 4) * 32 for k in range(K // 16)]
    offs_b = [(k // 4) * (N // 8) * 1024 + (k % 4) * 32 for k in range(K // 16)]
    d = run(probe, 0, sw128_k(gb), sw128_k(cb), None, N, K, (16, 1024, 1, 0, offs_a), (16, 1024, 1, 0, offs_b))
    np.testing.assert_allclose(d, g @ c.T, rtol=1e-5, atol=1e-3)


def test_m64_row_mapping(probe):
    """Record where an M=64 accumulator lands in TMEM lanes (the fused Gram uses one for rows 128..)."""
    rng = np.random.default_rng(5)
    M, N, K = 64, 32, 16
    ab, a = bf16_bits(rng.normal(size=(M, K)))
    wb, w = bf16_bits(rng.normal(size=(N, K)))
    d = run(probe, 0, blocked(ab), blocked(wb), None, N, K, (128, (K // 8) * 128, 0, 0, [0]),
            (128, (K // 8) * 128, 0, 0, [0]), M=64)
    ref = a @ w.T
    lanes = []
    for r in range(M):
        hit = [ln for ln in range(128) if np.allclose(d[ln], ref[r], rtol=1e-5, atol=1e-4)]
        lanes.append(hit[0] if hit else -1)
    print("M=64 row -> lane:", lanes)
    assert all(x >= 0 for x in lanes)
    assert lanes == list(range(64)) or lanes == [16 * (r // 16) * 2 + r % 16 for r in range(64)]
