"""The multi-rank path on the device: two processes share cuda:0 (gloo all_reduce on CUDA tensors).

Each rank runs the REAL fused chain kernels on its own shard -- an X-slab of one volume
(distributed.voxel_slab) or its own subjects (distributed.shard_range) -- then sums the LSC
gradients with distributed.allreduce_gradients, exactly the code bench.py runs over NCCL on
N GPUs.  The all-reduced dW / db and every rank's y / dx slab must equal the single-volume
result of the oracle (oracle/port.py) within the LSC tolerance (1e-4, north_star).  The ranks'
kernels never wait on one another (the only exchange is the host-side gloo all_reduce), so
sharing one GPU is safe.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port

pytestmark = pytest.mark.gpu

WORLD = 2
TOL = 1e-4
GRID = (9, 7, 6)


def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(nsub):
    from paper_1808_01517_b200.directions import unit_sphere_directions

    d = unit_sphere_directions(90)
    rng = np.random.default_rng(11)
    w = rng.normal(size=(3, 3, 6)) / 18.0
    b = rng.normal(size=3) * 0.1
    x = np.asarray(rng.uniform(0.1, 1.3, size=(nsub, 270, *GRID)), np.float32).astype(np.float64)
    dy = np.asarray(rng.normal(size=(nsub, 270, *GRID)), np.float32).astype(np.float64)
    return d, w, b, x, dy


def _worker(rank, port_no, mode, out):
    import paper_1808_01517_b200 as dl
    from paper_1808_01517_b200.distributed import allreduce_gradients, shard_range, voxel_slab

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        d, w, b, x, dy = _problem(1 if mode == "voxels" else 3)
        s2sh = dl.Signal2SH(8, d, lb_lambda=0.006).to(dev)
        lsc = dl.LocalSphericalConvolution(3, 3, 8, 8, d, [5], lb_lambda=0.006, angular_distance=np.pi / 5).to(dev)
        lsc.load_kernel(dl.LscKernel(w, b))
        chain = dl.SphericalChain(s2sh, lsc, dl.SH2Signal(8, d).to(dev))
        xt = torch.tensor(x, dtype=torch.float32, device=dev)
        dyt = torch.tensor(dy, dtype=torch.float32, device=dev)
        if mode == "voxels":
            xt, dyt = voxel_slab(xt, rank, WORLD), voxel_slab(dyt, rank, WORLD)
        else:
            lo, hi = shard_range(x.shape[0], rank, WORLD)
            xt, dyt = xt[lo:hi].contiguous(), dyt[lo:hi].contiguous()
        xt.requires_grad_(True)
        y = chain(xt)
        y.backward(dyt)
        params = list(lsc.parameters())
        allreduce_gradients(params)   # gloo on CUDA tensors
        torch.cuda.synchronize()
        out[rank] = (y.detach().double().cpu().numpy(), xt.grad.double().cpu().numpy(),
                     lsc.sconv.weight.grad.double().cpu().numpy()[:, :, 0, :], lsc.sconv.bias.grad.double().cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["voxels", "subjects"])
def test_sharded_chain_allreduce_matches_full_volume(mode):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1808_01517_b200._build import build_library

    build_library()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(_free_port(), mode, out), nprocs=WORLD, join=True)
    d, w, b, x, dy = _problem(1 if mode == "voxels" else 3)
    M, _, _ = port.fit_operator(d, 8, 0.006)
    geo = port.lsc_geometry(d, [5], np.pi / 5, 8, 8, 0.006)
    Bt = port.eval_basis(d, 8)
    wq = np.asarray(w, np.float32).astype(np.float64)
    bq = np.asarray(b, np.float32).astype(np.float64)
    y_ref = port.chain_forward(x, M, geo, wq, bq, Bt, 3)
    dx_ref, dW_ref, db_ref = port.chain_backward(x, dy, M, geo, wq, Bt, 3)
    axis = 2 if mode == "voxels" else 0
    y = np.concatenate([out[r][0] for r in range(WORLD)], axis=axis)
    dx = np.concatenate([out[r][1] for r in range(WORLD)], axis=axis)
    assert port.rel_err(y, y_ref) <= TOL
    assert port.rel_err(dx, dx_ref) <= TOL
    for r in range(WORLD):   # every rank holds the all-reduced (whole-volume) gradient
        assert port.rel_err(out[r][2], dW_ref) <= TOL
        assert port.rel_err(out[r][3], db_ref) <= TOL
    np.testing.assert_array_equal(out[0][2], out[1][2])
