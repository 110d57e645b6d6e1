"""Microbenchmark: tcgen05.ld.32x32b.x16 throughput of 12 warps while warp 0 streams MMAs (85 TS, 86 SS) or
TMEM stores (87), versus alone (81)."""
import ctypes, subprocess
out = "/tmp/mma_rate.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
                "-fPIC", "-o", out, "tests/cuda/mma_rate.cu"], check=True)
lib = ctypes.CDLL(out)
res = (ctypes.c_longlong * 2)()
cyc = 400000
for mode, N in ((81, 48), (85, 48), (85, 144), (85, 256), (86, 48), (86, 144), (87, 48)):
    st = lib.mma_rate(mode, N, cyc, res, 320, 12)
    n = res[1]
    extra = f", warp 0: {res[0]} {'MMA groups of 16' if mode in (85, 86) else 'stores'}" if mode >= 85 else ""
    print(f"mode {mode} N={N:3d}: {cyc / max(n, 1):7.1f} cyc/load/warp, {12 * n * 16 * 128 / cyc:7.1f} B/cyc{extra}"
          f" st={st}")
