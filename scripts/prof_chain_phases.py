"""Debug: per-role phase timestamps of CTA 0 in the forward chain kernel (dl_debug_chain_prof).

Prints, for tiles 2..5, every recorded event (role, event id) as cycles since tile 2's first event.
chain3v events: role 1: 0 CONV waits d1, 1 d1 ready, 2 D1 converted, 3 d2 ready, 8+2o OUT sees d3(o),
9+2o OUT drained d3(o); role 2 (stage-2/3 issuer): 0 tile start, 1 stage 2 done, 2+2o / 3+2o stage-3 group o
start / done; roles 0 / 3 (CONV warps 0 / 1 of quadrant 0): D2 item j: j start, 10+j converted, 20+j handed
over; roles 5 / 6: the same for D1 items; role 4 (stage-1 issuer): 3g group g, 3g+1 its D1 buffer free,
10+k IN item k full.
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
nograd = len(sys.argv) > 1 and sys.argv[1] == 'nograd'   # no weight gradient: no c_mid stores
ctx = torch.no_grad() if nograd else torch.enable_grad()
with ctx:
    for _ in range(2):
        y = chain(x)
    torch.cuda.synchronize()
    lib.dl_debug_chain_prof(ctypes.c_void_p(buf.data_ptr()))
    y = chain(x)
    torch.cuda.synchronize()
    lib.dl_debug_chain_prof(None)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(5):
        y = chain(x)
    ev1.record()
torch.cuda.synchronize()
print(f'forward {ev0.elapsed_time(ev1) / 5:.3f} ms per call (nograd={nograd})')
torch.cuda.synchronize()
lib.dl_debug_chain_prof(None)
b = buf.cpu().numpy()[:2048].reshape(8, 8, 32)
t0 = min(v for v in b[2].ravel() if v)
for it in range(2, 6):
    ev = sorted((int(b[it, r, e]) - t0, r, e) for r in range(8) for e in range(32) if b[it, r, e])
    print(f'tile {it}: ' + ' '.join(f'{r}.{e}@{t}' for t, r, e in ev))
