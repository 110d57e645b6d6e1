"""Microbenchmark: tcgen05.ld throughput with no MMA running, by load width and warp count (mma_rate.cu 80-84)."""
import ctypes, subprocess
out = "/tmp/mma_rate.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
                "-fPIC", "-o", out, "tests/cuda/mma_rate.cu"], check=True)
lib = ctypes.CDLL(out)
res = (ctypes.c_longlong * 2)()
cols = {80: 8, 81: 16, 82: 32, 83: 16, 84: 32}
for mode in (80, 81, 82, 83, 84):
    for nw in (1, 4, 8, 16):
        cyc = 400000
        st = lib.mma_rate(mode, 48, cyc, res, 0, nw)
        n = res[1]
        print(f"mode {mode} (x{cols[mode]}) warps {nw:2d}: {cyc / max(n, 1):7.1f} cyc/load/warp, "
              f"{nw * n * cols[mode] * 128 / cyc:7.1f} B/cyc st={st}")
