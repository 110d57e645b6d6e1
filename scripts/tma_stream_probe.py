"""Microbenchmark: channel-pair TMA read (and read + row-segment write) bandwidth by row count and consumer count."""
import ctypes, subprocess, torch
out = "/tmp/tma_stream.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
                "-fPIC", "-o", out, "tests/cuda/tma_stream.cu"], check=True)
lib = ctypes.CDLL(out)
lib.tma_stream.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
lib.tma_stream_rw.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
nvox = 3658350
x = torch.randn(288 * nvox, device="cuda"); y = torch.empty(288 * nvox, device="cuda")
ms = ctypes.c_float()
for rows in (144, 288):
    lib.tma_stream(ctypes.c_void_p(x.data_ptr()), nvox, rows, 128, 8, 1, ctypes.byref(ms))
    gb = rows * nvox * 4 / 1e9
    print(f"reads only, 1 consumer warp,  rows={rows}: {ms.value:.3f} ms {gb/ms.value:.2f} TB/s")
    lib.tma_stream_rw(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), nvox, rows, 8, 0, ctypes.byref(ms))
    print(f"reads only, 4 consumer warps, rows={rows}: {ms.value:.3f} ms {gb/ms.value:.2f} TB/s")
    lib.tma_stream_rw(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), nvox, rows, 8, -1, ctypes.byref(ms))
    print(f"reads only, 4 warps, LDS.128 row-wise, rows={rows}: {ms.value:.3f} ms {gb/ms.value:.2f} TB/s")
    lib.tma_stream_rw(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), nvox, rows, 8, 16, ctypes.byref(ms))
    print(f"read+write,  4 consumer warps, rows={rows}: {ms.value:.3f} ms {2*gb/ms.value:.2f} TB/s")
