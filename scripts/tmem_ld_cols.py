"""Microbenchmark: tcgen05.ld.32x32b.x16 throughput (16 warps, no MMA) by TMEM column offset."""
import ctypes, subprocess
out = "/tmp/mma_rate.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
                "-fPIC", "-o", out, "tests/cuda/mma_rate.cu"], check=True)
lib = ctypes.CDLL(out)
res = (ctypes.c_longlong * 2)()
for col in (0, 64, 128, 192, 256, 320, 384, 448, 480, 496):
    for nw in (1, 12):
        cyc = 400000
        st = lib.mma_rate(81, 48, cyc, res, col, nw)
        n = res[1]
        print(f"col {col:3d} warps {nw:2d}: {cyc / max(n, 1):7.1f} cyc/load/warp, {nw * n * 16 * 128 / cyc:7.1f} B/cyc st={st}")
