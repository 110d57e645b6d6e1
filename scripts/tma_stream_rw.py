"""Microbenchmark: the chain kernel's HBM pattern without compute (tests/cuda/tma_stream.cu stream_rw_k):
TMA channel-pair reads of 288 rows x 128-voxel tiles, thread-per-voxel 128-byte row-segment stores of 270 rows,
one persistent CTA per SM -- how fast the memory system moves the chain's 7.9 GB in this shape."""
import ctypes, subprocess
import torch
out = "/tmp/tma_stream.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
                "-fPIC", "-o", out, "tests/cuda/tma_stream.cu"], check=True)
lib = ctypes.CDLL(out)
lib.tma_stream_rw.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                              ctypes.POINTER(ctypes.c_float)]
nvox, rows = 3658350, 288
x = torch.randn(rows * nvox, device="cuda")
y = torch.empty(rows * nvox, device="cuda")
ms = ctypes.c_float()
for NS in (4, 8, 12):
    for wrows in (0, 16):
        st = lib.tma_stream_rw(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), nvox, rows, NS, wrows,
                               ctypes.byref(ms))
        gb = rows * nvox * 4 * (1 + wrows / 16) / 1e9
        print(f"NS={NS:2d} writes={'yes' if wrows else 'no '}: {ms.value:.3f} ms  {gb:.2f} GB  {gb / ms.value * 1e3:.0f} GB/s  st={st}")
