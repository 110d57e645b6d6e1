"""Microbenchmark: TMA channel-pair streaming bandwidth (tests/cuda/tma_stream.cu)."""
import ctypes, subprocess
import torch
out = "/tmp/tma_stream.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
                "-fPIC", "-o", out, "tests/cuda/tma_stream.cu"], check=True)
lib = ctypes.CDLL(out)
lib.tma_stream.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                           ctypes.POINTER(ctypes.c_float)]
nvox, rows = 3658350, 144
x = torch.randn(rows * nvox, device="cuda")
ms = ctypes.c_float()
for W in (64, 128, 256):
    for NS in (4, 8, 16):
        if 1024 + NS * 16 * (W + 4) * 4 > 227 * 1024:
            continue
        st = lib.tma_stream(ctypes.c_void_p(x.data_ptr()), nvox, rows, W, NS, 1, ctypes.byref(ms))
        gb = rows * nvox * 4 / 1e9
        print(f"W={W:3d} NS={NS:2d} in-flight={NS * 16 * (W + 4) * 4 / 1024:6.1f} KB: {ms.value:.3f} ms  {gb / ms.value:.0f} GB/s  st={st}")
