"""Microbenchmark cycles per tcgen05.mma issue (test-only probe, tests/cuda/mma_rate.cu)."""
import ctypes, subprocess, sys
out = "/tmp/mma_rate.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
                "-fPIC", "-o", out, "tests/cuda/mma_rate.cu"], check=True)
lib = ctypes.CDLL(out)
res = (ctypes.c_longlong * 2)()
for N in (48, 144):
    for mode in (30, 33, 34, 37):
        iters = 4000
        st = lib.mma_rate(mode, N, iters, res, 0, 256)
        print(f"N={N:3d} TS traffic={['none', 'ld', 'st', 'ld+st', 'smem', 'ld+smem', 'st+smem', 'ld+st+smem'][mode - 30]:10s}: "
              f"{res[0] / iters:7.1f} cyc/mma (ideal {N / 2:.0f}) st={st}")

print("kernel-like B images (K-major SBO=Kc/8*128 / MN-major)")
for N in (48, 96, 144):
    for mode in (50, 51):
        iters = 6000
        st = lib.mma_rate(mode, N, iters, res, 0, 256)
        print(f"N={N:3d} {'Kmaj' if mode == 50 else 'MNmaj'}: {res[0] / iters:7.1f} cyc/mma (ideal {N / 2:.0f}) st={st}")
