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

print("issue cost under contention (busy warps), registers-carried vs recomputed descriptors")
for N in (48, 144):
    for busy in (0, 7, 15, 27):
        r = []
        for mode in (60, 61):
            iters = 6000
            st = lib.mma_rate(mode, N, iters, res, 0, 256 | (busy << 16))
            r.append(res[0] / iters)
        print(f"N={N:3d} busy warps={busy:2d}: carried {r[0]:6.1f}  recomputed {r[1]:6.1f} cyc/mma (ideal {N / 2:.0f})")

for mode in (70, 71):
    iters = 54 * 200
    st = lib.mma_rate(mode, 144, iters, res, 0, 0)
    print(f"stage-2 pattern ({'3 images' if mode == 70 else 'same image'}): {res[0] / iters:6.1f} cyc/mma (ideal 72) st={st}")
