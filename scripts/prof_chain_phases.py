"""Debug: per-role phase timestamps of CTA 0 in the forward chain kernel (dl_debug_chain_prof).

Prints, for tiles 2..5, every recorded event (role, event id) as cycles since tile 2's first event.
chain3v events (role 1): 0 CONV waits d1, 1 d1 ready, 2 D1 converted, 3 d2 ready, 4+o A3(o) converted,
8+2o OUT sees d3(o), 9+2o OUT drained d3(o).
"""
import ctypes
import sys

import torch

sys.path.insert(0, '/root/repo')
import bench  # noqa: E402
from paper_1808_01517_b200 import _lib  # noqa: E402

dev = torch.device('cuda:0')
dirs, lsc, chain = bench.build_model(dev)
x, dy = bench.synth_inputs(dirs, (145, 174, 145), 0, dev)
buf = torch.zeros(4096, dtype=torch.int64, device=dev)
lib = _lib.load()
for _ in range(2):
    y = chain(x)
torch.cuda.synchronize()
lib.dl_debug_chain_prof(ctypes.c_void_p(buf.data_ptr()))
y = chain(x)
torch.cuda.synchronize()
lib.dl_debug_chain_prof(None)
b = buf.cpu().numpy()[:1024].reshape(8, 4, 32)
t0 = min(v for v in b[2].ravel() if v)
for it in range(2, 6):
    ev = sorted((int(b[it, r, e]) - t0, r, e) for r in range(4) for e in range(32) if b[it, r, e])
    print(f'tile {it}: ' + ' '.join(f'{r}.{e}@{t}' for t, r, e in ev))
