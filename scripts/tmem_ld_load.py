"""Microbenchmark: tcgen05.ld (x16) throughput of 12 warps while one warp streams TS MMAs (tests/cuda/mma_rate.cu
modes 30/31).  Prints MMA cycles and loads per warp completed meanwhile -> bytes/cycle of TMEM reads."""
import ctypes, subprocess
out = "/tmp/mma_rate.so"
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared", "-Xcompiler",
                "-fPIC", "-o", out, "tests/cuda/mma_rate.cu"], check=True)
lib = ctypes.CDLL(out)
res = (ctypes.c_longlong * 2)()
for N in (48, 144, 256):
  for ss in (0, 1, 2):
    for mode in (30, 31, 32):
        iters = 20000
        st = lib.mma_rate(mode, N, iters, res, ss << 16, 256)
        cyc = res[0]
        n = res[1] if mode in (31, 32) else 0
        # warp 4 did n loads of 2 KB; 12 loader warps (4..15) do about the same
        print(f"{['TS', 'SS', 'no-MMA'][ss]} N={N:3d} mode={mode}: {cyc / iters:6.1f} cyc/mma; loads/warp {n}; "
              f"TMEM ld ~{12 * n * 2048 / cyc:6.1f} B/cyc (12 warps) st={st}")
