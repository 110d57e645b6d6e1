"""Debug: per-role phase timestamps of CTA 0 in the forward chain3 kernel (dl_debug_chain_prof)."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import bench
from paper_1808_01517_b200 import _lib

dev = torch.device('cuda:0')
dirs, lsc, chain = bench.build_model(dev)
x, dy = bench.synth_inputs(dirs, (145, 174, 145), 0, dev)
buf = torch.zeros(2048, dtype=torch.int64, device=dev)
lib = _lib.load()
for _ in range(2):
    y = chain(x)
torch.cuda.synchronize()
lib.dl_debug_chain_prof(ctypes.c_void_p(buf.data_ptr()))
y = chain(x)
torch.cuda.synchronize()
lib.dl_debug_chain_prof(None)
allb = buf.cpu().numpy()
print('IN phase cycles (issue, data, a_empty, split, st+arrive):', allb[1000:1005])
b = allb[:1024].view().reshape(8, 4, 32)
t0 = b[0, 0, 0]
names = {
    0: {0: 'tile', 1: 'g0', 2: 'g1', 3: 'g2'},
    1: {0: 'w.d1', 1: 'd1', 2: 'A2done', 3: 'u', 4: 'A3_0', 5: 'y0', 6: 'st0', 7: 'A3_1', 8: 'y1', 9: 'st1', 10: 'A3_2', 11: 'y2', 12: 'st2'},
    2: {1: 's1g0', 2: 's1g1', 3: 's1g2', 8: 's2', 9: 'ac', 10: 's3o0', 11: 'au0', 12: 's3o1', 13: 'au1', 14: 's3o2', 15: 'au2'},
    3: {0: 'tile'},
}
for it in range(2, 5):
    print('tile', it)
    for r, nm in zip(range(4), ['IN ', 'MID', 'MMA', 'LD ']):
        print('  ', nm, ' '.join(f"{names[r][k]}={(b[it, r, k] - t0)}" for k in sorted(names[r]) if b[it, r, k]))
