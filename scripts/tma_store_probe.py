"""Run tests/cuda/tma_store_probe.cu: TMA store + load of a box at 16-byte aligned and 8-byte aligned starts."""
import ctypes, subprocess
import numpy as np
out = "/tmp/tma_store_probe.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
                "-fPIC", "-o", out, "tests/cuda/tma_store_probe.cu", "-lcuda"], check=True)
lib = ctypes.CDLL(out)
nvox = 1002
for u0 in (32, nvox + 32, nvox + 30, 33):
    g = np.zeros(16 * nvox, np.float32)
    back = np.zeros(256, np.float32)
    st = lib.tma_store_probe(ctypes.c_int64(nvox), u0, g.ctypes.data_as(ctypes.c_void_p), back.ctypes.data_as(ctypes.c_void_p))
    pairs = g.reshape(8, 2 * nvox)
    want = 1000 + np.arange(256, dtype=np.float32).reshape(8, 32)
    inbox = pairs[:, u0:u0 + 32]
    written = ~np.isnan(pairs)
    outside = written.sum() - written[:, u0:u0 + 32].sum()
    print(f"u0={u0} (byte offset mod 16 = {(u0 * 4) % 16}): status {st}, box ok {np.array_equal(inbox, want)}, "
          f"writes outside box {outside}, load-back ok {np.array_equal(back.reshape(8, 32), want)}")
