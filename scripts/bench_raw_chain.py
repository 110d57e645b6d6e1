"""SURVEY.md 8(f) row 1 measured: b0 normalisation fused into the chain kernel vs the two-pass pipeline.

An HCP-sized int16 acquisition (145 x 174 x 145 voxels, 18 b0 + 3 x 90 diffusion volumes interleaved, x-fastest
like a NIfTI file's voxel bytes), already on the device.  Times, with CUDA events (median of `reps` after 2
warm-ups):
  two-pass   ingest.normalize_b0 (fp32 (1, 270, X, Y, Z) volume in HBM) -> SphericalChain forward (fp16 pass)
  fused      ingest.chain_from_raw: b0 factors (dl_b0_voxel_scale_f32) + the chain kernel reading the int16
             volumes with the normalisation in its input role (dl_chain_fwd_raw_f32, 3-term bf16 pass)
and checks the two agree (max rel err).  Prints one JSON line (committed as profiles/r02_raw_chain.json).
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1808_01517_b200 as dl  # noqa: E402
from paper_1808_01517_b200 import dwio  # noqa: E402


def main(reps=10, save=False):
    dev = torch.device("cuda:0")
    X, Y, Z = bench.GRID
    nvox = X * Y * Z
    dirs, s2sh, lscs, sh2s = bench.chain_modules(dev)
    chain = dl.SphericalChain(s2sh, lscs[0], sh2s)
    n_b0, N = 18, 90
    # interleave: a b0 every 16 volumes, shells 1000 / 2000 / 3000 in turn
    layout = []
    for i in range(3 * N):
        if i % 15 == 0 and len([v for v in layout if v < 0]) < n_b0:
            layout.append(-1)
        layout.append(i)
    while len([v for v in layout if v < 0]) < n_b0:
        layout.append(-1)
    V = len(layout)
    bvals = np.zeros(V)
    for j, v in enumerate(layout):
        bvals[j] = 0.0 if v < 0 else 1000.0 * (1 + v % 3)
    dirs_all = np.zeros((V, 3))
    for j, v in enumerate(layout):
        if v >= 0:
            dirs_all[j] = dirs[v // 3]
    shells = tuple(dwio.Shell(1000.0 * (s + 1), np.array([j for j, v in enumerate(layout) if v >= 0 and v % 3 == s]))
                   for s in range(3))
    scheme = dwio.GradientScheme(dirs_all, bvals, np.array([j for j, v in enumerate(layout) if v < 0]), shells,
                                 dwio.B0_THRESHOLD)
    # synthetic signal: the bench's band-limited volume times a b0 image, quantised to int16
    x = bench.synth_signal(dirs, bench.GRID, 0, dev)                      # (1, 270, X, Y, Z)
    gen = torch.Generator(device=dev).manual_seed(5)
    b0img = 1500.0 + 500.0 * torch.rand((X, Y, Z), generator=gen, device=dev)
    raw = torch.empty((V, Z, Y, X), dtype=torch.int16, device=dev)     # stored order: x fastest, volumes slowest
    for j, v in enumerate(layout):
        val = b0img if v < 0 else x[0, (v % 3) * N + v // 3] * b0img
        raw[j] = val.round().clamp(-32768, 32767).to(torch.int16).permute(2, 1, 0)
    del x
    stored = raw.permute(3, 2, 1, 0)                                    # (X, Y, Z, V) view, strides (1, X, XY, XYZ)

    def two_pass():
        vol, _ = dl.normalize_b0(stored, scheme, device=dev)
        with torch.no_grad():
            return chain(vol.data)

    def fused():
        return dl.chain_from_raw(chain, stored, scheme, device=dev)[0]

    res = {}
    for name, fn in (("two_pass", two_pass), ("fused", fused)):
        for _ in range(2):
            out = fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name] = (statistics.median(ts), out)
    a, b = res["two_pass"][1].double(), res["fused"][1].double()
    err = float((a - b).abs().max() / a.abs().max())
    line = {"what": "load->chain of an HCP-sized int16 acquisition (145x174x145, 18 b0 + 270 DW volumes, on device)",
            "two_pass_ms": res["two_pass"][0], "fused_ms": res["fused"][0],
            "voxels_per_s_fused": nvox / (res["fused"][0] / 1e3), "rel_err_fused_vs_two_pass": err,
            "raw_bytes": int(raw.numel() * 2)}
    print(json.dumps(line))
    if save:
        with open(os.path.join(ROOT, "profiles", "r02_raw_chain.json"), "w") as f:
            json.dump(line, f, indent=1)


if __name__ == "__main__":
    main(save="--save" in sys.argv)
