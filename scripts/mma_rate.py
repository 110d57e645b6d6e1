"""Microbenchmark cycles per tcgen05.mma issue (test-only probe, tests/cuda/mma_rate.cu)."""
import ctypes, subprocess, sys
out = "/tmp/mma_rate.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
                "-fPIC", "-o", out, "tests/cuda/mma_rate.cu"], check=True)
lib = ctypes.CDLL(out)
res = (ctypes.c_longlong * 2)()
for N in (48, 144):
    for v in range(8):
        iters = 6000
        st = lib.mma_rate(40 + v, N, iters, res, 0, 256)
        print(f"N={N:3d} kstep6 commit={v & 1} fence={(v >> 1) & 1} poll={(v >> 2) & 1}: issue {res[0] / iters:6.1f} "
              f"complete {res[1] / iters:6.1f} cyc/mma (ideal {N / 2:.0f}) st={st}")
