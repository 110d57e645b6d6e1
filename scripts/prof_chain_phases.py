import ctypes, numpy as np, torch, math, sys
sys.path.insert(0, '/root/repo')
import bench
from paper_1808_01517_b200 import _lib
dev = torch.device('cuda:0')
dirs, lsc, chain = bench.build_model(dev)
x, dy = bench.synth_inputs(dirs, (145,174,145), 0, dev)
buf = torch.zeros(8*2*32, dtype=torch.int64, device=dev)
lib = _lib.load()
for _ in range(2): y = chain(x)
torch.cuda.synchronize()
lib.dl_debug_chain_prof(ctypes.c_void_p(buf.data_ptr()))
y = chain(x)
torch.cuda.synchronize()
lib.dl_debug_chain_prof(None)
b = buf.view(8, 2, 32).cpu().numpy()
t0 = b[0,0,0]
names = {0:'tile',1:'g0 start',2:'g0 arrive',3:'g1 start',4:'g1 arr',5:'g2 start',6:'g2 arr',8:'c_full',9:'ac arr',10:'u_full',11:'au0',12:'y0',13:'st0',14:'au1',15:'y1',16:'st1',17:'au2',18:'y2',19:'st2'}
mnames = {1:'w ax0',2:'got ax0',3:'w ax1',4:'got ax1',5:'w ax2',6:'got ax2',8:'w ac',9:'got ac',10:'iss2 done',11:'got au0',12:'iss y0',14:'got au1',15:'iss y1',17:'got au2',18:'iss y2'}
for it in range(4):
    print('tile', it)
    print('  E  :', ' '.join(f"{names[k]}={(b[it,0,k]-t0)}" for k in sorted(names) if b[it,0,k]))
    print('  MMA:', ' '.join(f"{mnames[k]}={(b[it,1,k]-t0)}" for k in sorted(mnames) if b[it,1,k]))
