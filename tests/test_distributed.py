"""Multi-process (gloo, world_size 2, CPU) tests of the subject sharding and the LSC gradient all-reduce.

The multi-GPU path (bench.py --gpus N) shards subjects across ranks with no data-path collective and
sums the LSC parameter gradients with one bucketed all_reduce (paper_1808_01517_b200/distributed.py).
Here the per-rank gradients come from the oracle (the checker), so the test covers exactly the host
logic that runs on NCCL on the GPU box: shard -> local backward -> all_reduce == full-batch backward.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port
from paper_1808_01517_b200.distributed import allreduce_gradients, max_over_ranks, shard_range

WORLD = 2


def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    rng = np.random.default_rng(7)
    d = rng.normal(size=(30, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    M, _, _ = port.fit_operator(d, 4, 0.006)
    geo = port.lsc_geometry(d, [5], np.pi / 5, 4, 4, 0.006)
    Bt = port.eval_basis(d, 4)
    K = geo["K"]
    w = rng.normal(size=(2, 2, K)) * 0.3
    x = rng.normal(size=(5, 2 * 30, 3, 2, 2))       # 5 subjects: an uneven 3/2 split
    dy = rng.normal(size=(5, 2 * 30, 3, 2, 2))
    return x, dy, M, geo, w, Bt


def _worker(rank, port_no, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        x, dy, M, geo, w, Bt = _problem()
        lo, hi = shard_range(x.shape[0], rank, WORLD)
        _, dW, db = port.chain_backward(x[lo:hi], dy[lo:hi], M, geo, w, Bt, 2)
        weight = torch.nn.Parameter(torch.zeros(w.shape, dtype=torch.float64))
        bias = torch.nn.Parameter(torch.zeros(2, dtype=torch.float64))
        weight.grad = torch.from_numpy(np.ascontiguousarray(dW))
        bias.grad = torch.from_numpy(np.ascontiguousarray(db))
        nbytes = allreduce_gradients([weight, bias])
        slowest = max_over_ranks(float(rank + 1))
        out[rank] = (lo, hi, weight.grad.numpy().copy(), bias.grad.numpy().copy(), nbytes, slowest)
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions_exactly():
    for n in (0, 1, 5, 7, 148, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_allreduce_single_process_is_identity():
    p = torch.nn.Parameter(torch.ones(3))
    p.grad = torch.arange(3.0)
    assert allreduce_gradients([p], scale=2.0) == 12
    assert torch.equal(p.grad, torch.arange(3.0) * 2)


def test_sharded_backward_allreduce_equals_full_batch():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(_free_port(), out), nprocs=WORLD, join=True)
    x, dy, M, geo, w, Bt = _problem()
    _, dW_full, db_full = port.chain_backward(x, dy, M, geo, w, Bt, 2)
    spans = sorted((out[r][0], out[r][1]) for r in range(WORLD))
    assert spans == [(0, 3), (3, 5)]
    for r in range(WORLD):
        _, _, dW, db, nbytes, slowest = out[r]
        assert nbytes == (dW_full.size + db_full.size) * 8   # one bucket
        assert slowest == float(WORLD)                        # max over ranks
        np.testing.assert_allclose(dW, dW_full, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(db, db_full, rtol=1e-12, atol=1e-12)


def test_voxel_slabs_partition_the_volume():
    from paper_1808_01517_b200.distributed import slab_range, voxel_slab

    x = torch.arange(2 * 3 * 7 * 2 * 2, dtype=torch.float32).view(2, 3, 7, 2, 2)
    for world in (1, 2, 3, 4, 8):
        slabs = [voxel_slab(x, r, world) for r in range(world)]
        assert all(s.is_contiguous() for s in slabs)
        assert torch.equal(torch.cat(slabs, dim=2), x)
        assert [slab_range(x, r, world) for r in range(world)] == [shard_range(7, r, world) for r in range(world)]
    with pytest.raises(ValueError):
        slab_range(x[0], 0, 2)


def _slab_worker(rank, port_no, out):
    """One X-slab of ONE volume per rank: local backward on the slab, then the bucketed all_reduce."""
    from paper_1808_01517_b200.distributed import voxel_slab

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        x, dy, M, geo, w, Bt = _problem()
        xs = voxel_slab(torch.from_numpy(x[:1]), rank, WORLD).numpy()
        dys = voxel_slab(torch.from_numpy(dy[:1]), rank, WORLD).numpy()
        _, dW, db = port.chain_backward(xs, dys, M, geo, w, Bt, 2)
        weight = torch.nn.Parameter(torch.zeros(w.shape, dtype=torch.float64))
        bias = torch.nn.Parameter(torch.zeros(2, dtype=torch.float64))
        weight.grad = torch.from_numpy(np.ascontiguousarray(dW))
        bias.grad = torch.from_numpy(np.ascontiguousarray(db))
        allreduce_gradients([weight, bias])
        out[rank] = (xs.shape[2], weight.grad.numpy().copy(), bias.grad.numpy().copy())
    finally:
        dist.destroy_process_group()


def test_voxel_slab_backward_allreduce_equals_full_volume():
    """Single-volume sharding: per-slab gradients summed over ranks == the volume's gradient."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_slab_worker, args=(_free_port(), out), nprocs=WORLD, join=True)
    x, dy, M, geo, w, Bt = _problem()
    _, dW_full, db_full = port.chain_backward(x[:1], dy[:1], M, geo, w, Bt, 2)
    assert sorted(out[r][0] for r in range(WORLD)) == [1, 2]
    for r in range(WORLD):
        np.testing.assert_allclose(out[r][1], dW_full, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(out[r][2], db_full, rtol=1e-12, atol=1e-12)
