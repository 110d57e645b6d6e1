"""Throughput of the ingest kernel (dl_normalize_b0_f32) on an HCP-sized raw acquisition.

145 x 174 x 145 voxels, 288 int16 volumes stored x-fastest (a NIfTI file's own bytes: 18 b0 + 3 x 90 shell
volumes), normalised into (1, 270, 145, 174, 145) fp32.  Algorithmic bytes per launch: b0 volumes read once
for the mean, the 270 shell volumes read once, the output written once, the float64 mean written and read
back once.  Prints one JSON line with GB/s and the fraction of MEASURED_PEAKS hbm_gbs.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_01517_b200 as dl  # noqa: E402
from paper_1808_01517_b200 import dwio  # noqa: E402

X, Y, Z = 145, 174, 145
bvals = np.array([0.0] * 18 + [1000.0] * 90 + [2000.0] * 90 + [3000.0] * 90)
rng = np.random.default_rng(0)
order = rng.permutation(bvals.size)
bvals = bvals[order]
dev = torch.device("cuda:0")
V = bvals.size
stored = torch.randint(100, 4000, (V, Z, Y, X), dtype=torch.int16, device=dev)   # x fastest, volume slowest
raw = stored.permute(3, 2, 1, 0)                                                   # (X, Y, Z, V) view
vol, mask = dl.normalize_b0(raw, bvals, device=dev)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record()
for _ in range(reps):
    vol, mask = dl.normalize_b0(raw, bvals, device=dev)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
nvox = X * Y * Z
nbytes = nvox * (18 * 2 + 270 * 2 + 270 * 4 + 8 + 8 + 1)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
print(json.dumps({"kernel": "dl_normalize_b0_f32 (int16 x-fastest -> fp32 channel-major)", "ms": ms,
                  "algorithmic_bytes": nbytes, "gbs": nbytes / ms / 1e6, "frac_of_hbm_peak": nbytes / ms / 1e6 / peak,
                  "note": "per call incl. index uploads and workspace allocation"}))
