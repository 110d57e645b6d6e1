"""Microbenchmark cycles per tcgen05.mma issue (test-only probe, tests/cuda/mma_rate.cu)."""
import ctypes, subprocess, sys
out = "/tmp/mma_rate.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
                "-fPIC", "-o", out, "tests/cuda/mma_rate.cu"], check=True)
lib = ctypes.CDLL(out)
res = (ctypes.c_longlong * 2)()
NAMES = {0: 'SS', 1: 'TS', 10: 'SS-elect', 11: 'TS-elect', 12: 'SS-elect-x4acc', 21: '1warp', 22: '2warps', 24: '4warps'}
for mode in (10, 21, 22, 24):
    for N in (16, 48, 96, 128):
        if mode >= 20 and (mode - 20) * N > 512: continue
        iters = 2000
        st = lib.mma_rate(mode, N, iters, res)
        print(f"{NAMES[mode]} N={N:3d}: issue {res[0] / iters:7.1f} cyc/mma, complete {res[1] / iters:7.1f} cyc/mma"
              f"  (ideal {128 * N / 256:.0f})  st={st}")
