#!/usr/bin/env python
"""Benchmark of the DELIMIT spherical-signal path on B200 (BASELINE.json configs).

    python bench.py [--config cfg4] [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1 without torchrun re-executes itself under `torch.distributed.run` (one rank per GPU,
NCCL); it fails loudly when fewer than N GPUs are visible.  Rank 0 prints ONE JSON line.

Configs (BASELINE.json configs[0..4]):
  cfg1  Signal2SH(8, 90 dirs) forward on (1, 90, 32, 32, 32)                          replicas
  cfg2  fused Signal2SH -> SH2Signal round trip fwd + bwd, (1, 270, 145, 174, 145)      subject per rank
  cfg3  LocalSphericalConvolution 1->1 fwd + bwd, (4, 45, 32, 32, 32)                   replicas
  cfg4  fused Signal2SH -> LSC 3->3 -> SH2Signal fwd + bwd, (1, 270, 145, 174, 145)     subject per rank
        (default; --shard voxels splits ONE subject into X-slabs across ranks instead)
  cfg5  Signal2SH -> 2 x LSC -> SH2Signal training step (fused MSE, SGD) on a global batch of 8
        HCP-sized subjects, 8 / N per rank, one bucketed NCCL all_reduce of the LSC gradients

Inputs are synthetic (phantom.py:77-88 band-limited signals + noise, N(0,1) upstream gradients) generated
on the device; every HCP-sized input (3.95 GB) exceeds the 126 MB L2, so no flush is needed there; the
32^3 configs flush L2 between timed steps.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "voxels/s fused Signal2SH→LSC→SH2Signal fwd+bwd; HBM GB/s % of peak; 1–8 GPU"
GRID = (145, 174, 145)
SHELLS, NDIR, ORDER, LAM = 3, 90, 8, 0.006
FALLBACK_HBM, FALLBACK_TF = 6650.0, 1590.0
NOMINAL_HBM = 8000.0
DTYPE_CHAIN = "f32 (fp16x2 split products with fp32 accumulation under delayed scaling; bf16x3 check pass)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("bf16_tflops", FALLBACK_TF)), "measured"
    except Exception:
        return FALLBACK_HBM, FALLBACK_TF, "fallback"


def ncu_traffic(kernel: str, key: str | None = None):
    """Per-launch DRAM bytes for `kernel` from the committed ncu capture (profiles/ncu_traffic.json), or another of
    its per-kernel tables (`key`, e.g. tensor_pipe_active_pct), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(kernel) if key is None else d.get(key, {}).get(kernel)
    except Exception:
        return None


def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args) -> None:
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run (or fail loudly)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus and args.dist_backend == "nccl":
        log(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, this box has {have}")
        sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    log("bench.py: launching", " ".join(cmd))
    os.execv(sys.executable, cmd)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw,power.limit,"
              "clocks.mem")

    def __init__(self, uuid: str | None):
        self.proc = None
        self.uuid = uuid

    def start(self):
        cmd = ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "20"]
        if self.uuid:
            cmd += ["-i", self.uuid]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception as exc:  # pragma: no cover
            log(f"clock sampling unavailable: {exc}")
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons, pw, plim, mem = [], None, set(), [], None, []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 9:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
            try:
                pw.append(float(parts[6]))
                plim = float(parts[7])
                mem.append(float(parts[8]))
            except ValueError:
                pass
        if not sm:
            return None
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        res = {"sm_mhz": statistics.median(loaded), "sm_min_mhz": min(loaded), "sm_max_mhz": mx,
               "reasons": sorted(reasons), "samples": len(sm)}
        if pw:
            res.update(power_w_median=statistics.median(pw), power_w_max=max(pw), power_limit_w=plim)
        if mem:
            res.update(mem_mhz=statistics.median(mem))
        return res


# ----------------------------------------------------------------------------- synthetic inputs
def synth_signal(dirs, grid, seed, dev, shells=SHELLS, batch=1):
    """Band-limited synthetic DWI (phantom.py:77-88 distribution) + N(0, 0.02^2) noise, on the device."""
    import torch

    from paper_1808_01517_b200.geometry import basis_degrees, eval_basis

    V = int(np.prod(grid))
    B = torch.tensor(eval_basis(dirs, ORDER), dtype=torch.float32, device=dev)
    l = torch.tensor(basis_degrees(ORDER), dtype=torch.float32, device=dev)
    amp = 0.9 / (1.0 + l * (l + 1.0) / 4.0)
    N = B.shape[0]
    x = torch.empty((batch, shells * N, V), dtype=torch.float32, device=dev)
    for b in range(batch):
        for s in range(shells):
            g = torch.Generator(device=dev).manual_seed(1000 + s + 7919 * seed + 104729 * b)
            coeffs = (torch.rand((B.shape[1], V), generator=g, device=dev) * 2 - 1) * amp[:, None]
            coeffs[0] = 2.0 * math.sqrt(math.pi)
            x[b, s * N:(s + 1) * N] = B @ coeffs
            x[b, s * N:(s + 1) * N] += 0.02 * torch.randn((N, V), generator=g, device=dev)
            del coeffs
    return x.view(batch, shells * N, *grid)


def synth_normal(shape, seed, dev):
    import torch

    g = torch.Generator(device=dev).manual_seed(2 + 7919 * seed)
    return torch.randn(shape, generator=g, device=dev)


def synth_inputs(dirs, grid, seed, dev):
    """(x, dy) of the cfg4 chain on one subject (kept for scripts/)."""
    x = synth_signal(dirs, grid, seed, dev)
    return x, synth_normal(x.shape, seed, dev)


def chain_modules(dev, layers=1):
    import paper_1808_01517_b200 as dl
    from paper_1808_01517_b200.directions import unit_sphere_directions

    dirs = unit_sphere_directions(NDIR)
    s2sh = dl.Signal2SH(ORDER, dirs, lb_lambda=LAM).to(dev)
    lscs = []
    for k in range(layers):
        lsc = dl.LocalSphericalConvolution(SHELLS, SHELLS, ORDER, ORDER, dirs, [5], lb_lambda=LAM,
                                           angular_distance=math.pi / 5).to(dev)
        w = np.random.default_rng(1 + k).normal(size=(SHELLS, SHELLS, 6)) / (SHELLS * 6)
        b = np.random.default_rng(1 + k).normal(size=SHELLS) * 0.1
        lsc.load_kernel(dl.LscKernel(w, b))
        lscs.append(lsc)
    sh2s = dl.SH2Signal(ORDER, dirs).to(dev)
    return dirs, s2sh, lscs, sh2s


def build_model(dev):
    """(dirs, lsc, chain) of cfg4 (kept for scripts/)."""
    import paper_1808_01517_b200 as dl

    dirs, s2sh, lscs, sh2s = chain_modules(dev)
    return dirs, lscs[0], dl.SphericalChain(s2sh, lscs[0], sh2s)


# ----------------------------------------------------------------------------- workloads
class Workload:
    """One config: `step()` is one pass of the path over this rank's inputs (already in HBM)."""

    name = ""
    metric = METRIC
    dtype = DTYPE_CHAIN
    scaling = "weak"
    graphed = True
    flush_l2 = False
    bytes_per_voxel = 0            # compulsory HBM bytes of the timed step per voxel
    dom = None                     # dominant kernel: (name, bytes per voxel per launch, ktimer slot or None)
    tensor_flops_per_voxel = 0.0   # MMA flops issued per voxel by the dominant kernel (0: SIMT)

    def __init__(self, args, dev, rank, world):
        self.args, self.dev, self.rank, self.world = args, dev, rank, world

    launch_groups = 1              # times the dominant kernel (and its companions) runs per step on a rank

    def voxels_per_step(self) -> int:   # all ranks
        raise NotImplementedError

    def voxels_per_launch(self) -> int:
        return self.V_local

    def step(self):
        raise NotImplementedError

    def phases(self):
        """Graph-capturable pieces of the step, in order (name, fn)."""
        return [("step", self.step)]

    def after_phases(self):
        """Host work after the graphed phases (e.g. the gradient all-reduce), not captured."""

    def e2e(self):
        return None

    def drop(self):
        """Release the last step's outputs and the autograd graph they keep alive (before graph capture: an
        AccumulateGrad node left from an eager step would tie the capture stream to the legacy stream)."""
        for attr in ("y", "u", "c", "loss"):
            if hasattr(self, attr):
                delattr(self, attr)
        for t in list(getattr(self, "params", [])) + [getattr(self, "x", None), getattr(self, "c_in", None)]:
            if t is not None and getattr(t, "grad", None) is not None:
                t.grad = None

    def cpu(self, steps, warmup):
        return None

    def config(self):
        return {}


def _l2_flush_buffer(dev):
    import torch

    return torch.empty(256 << 20, dtype=torch.uint8, device=dev)


class Cfg4(Workload):
    name = "cfg4"
    bytes_per_voxel = 5400          # x, y, dy, x-or-c, dx
    dom = ("chain_fwd", 2160, 0)
    # chain2h forward per 128-voxel tile: stage 1 3 shells x 6 K-steps x 3 products of 128x48x16, stage 2
    # 3 shells x 9 K-steps x 3 products of 128x96x16 (2 flops per MAC)
    tensor_flops_per_voxel = (3 * 6 * 3 * 128 * 48 * 16 * 2 + 3 * 9 * 3 * 128 * 96 * 16 * 2) / 128

    def __init__(self, args, dev, rank, world):
        super().__init__(args, dev, rank, world)
        import paper_1808_01517_b200 as dl

        self.shard = args.shard == "voxels" and world > 1
        self.scaling = "strong" if self.shard else "weak"
        grid = tuple(args.grid)
        self.V_subject = int(np.prod(grid))
        self.dirs, s2sh, lscs, sh2s = chain_modules(dev)
        self.lsc = lscs[0]
        self.chain = dl.SphericalChain(s2sh, self.lsc, sh2s)
        self.params = list(self.lsc.parameters())
        if self.shard:
            from paper_1808_01517_b200.distributed import voxel_slab

            x, dy = synth_inputs(self.dirs, grid, 0, dev)
            self.x, self.dy = voxel_slab(x, rank, world), voxel_slab(dy, rank, world)
            del x, dy
        else:
            self.x, self.dy = synth_inputs(self.dirs, grid, rank, dev)
        self.x.requires_grad_(True)
        self.V_local = self.x[0, 0].numel()

    def voxels_per_step(self):
        return self.V_subject if self.shard else self.world * self.V_subject

    def _fwd(self):
        self.x.grad = None
        for p in self.params:
            p.grad = None
        self.y = self.chain(self.x)

    def _bwd(self):
        self.y.backward(self.dy)

    def step(self):
        self._fwd()
        self._bwd()
        self.after_phases()

    def phases(self):
        return [("fwd", self._fwd), ("bwd", self._bwd)]

    def after_phases(self):
        if self.world > 1:
            from paper_1808_01517_b200.distributed import allreduce_gradients

            allreduce_gradients(self.params)

    def config(self):
        c = {"workload": "cfg4: fused Signal2SH(order 8, 90 dirs, lambda .006) -> LSC 3->3 ([5] ring, pi/5) -> "
                         "SH2Signal fwd+bwd (dx, dW, db), " +
                         ("one 145x174x145 subject split into X-slabs across ranks" if self.shard
                          else "one 145x174x145 subject per GPU"),
             "model": "SphericalChain", "global_batch": 1 if self.shard else self.world,
             "voxels_per_gpu": self.V_local, "channels": SHELLS * NDIR, "seq_len": None,
             "parallelism": (f"voxel-slab x{self.world}" if self.shard else f"dp{self.world} (subject-sharded)"),
             "l2": "no flush: each input (3.95 GB) exceeds the 126 MB L2"}
        return c

    def e2e(self):
        """The same step through the public module API from pinned host buffers: H2D of x and dy every step,
        D2H of the step's parameter gradients; a copy stream uploads step i+1's inputs while step i computes."""
        import torch

        dev, x, dy, chain, params = self.dev, self.x, self.dy, self.chain, self.params
        xh = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
        dyh = torch.empty(dy.shape, dtype=torch.float32, pin_memory=True)
        xh.copy_(x.detach())
        dyh.copy_(dy)
        wh = torch.empty(self.lsc.sconv.weight.shape, pin_memory=True)
        bh = torch.empty(self.lsc.sconv.bias.shape, pin_memory=True)
        cs = torch.cuda.Stream(device=dev)
        main = torch.cuda.current_stream(dev)
        xbuf = [torch.empty_like(x.detach()) for _ in range(2)]
        dybuf = [torch.empty_like(dy) for _ in range(2)]
        x_ready = [torch.cuda.Event() for _ in range(2)]
        dy_ready = [torch.cuda.Event() for _ in range(2)]
        freed = [torch.cuda.Event() for _ in range(2)]

        def upload(i, start=None):
            k = i % 2
            if start is not None:
                cs.wait_event(start)
            if i >= 2:
                cs.wait_event(freed[k])
            with torch.cuda.stream(cs):
                xbuf[k].copy_(xh, non_blocking=True)
                x_ready[k].record(cs)
                dybuf[k].copy_(dyh, non_blocking=True)
                dy_ready[k].record(cs)

        def e2e_step(i):
            k = i % 2
            for p in params:
                p.grad = None
            main.wait_event(x_ready[k])
            xd = xbuf[k].detach().requires_grad_(True)
            y = chain(xd)
            main.wait_event(dy_ready[k])
            y.backward(dybuf[k])
            del y
            freed[k].record(main)
            self.after_phases()
            wh.copy_(self.lsc.sconv.weight.grad, non_blocking=True)
            bh.copy_(self.lsc.sconv.bias.grad, non_blocking=True)

        upload(0)
        e2e_step(0)
        torch.cuda.synchronize()
        return _time_e2e(self, upload, e2e_step, int((xh.numel() + dyh.numel()) * 4), int((wh.numel() + bh.numel()) * 4),
                         "LSC dW, db (the step's parameter gradients)")

    def cpu(self, steps, warmup):
        from oracle import cpu_baseline as cb

        nvox = self.args.cpu_sample
        orc = cb.ChainOracle(self.dirs)
        x, dy = cb.synthetic_sample(self.dirs, nvox)
        w = np.random.default_rng(1).normal(size=(SHELLS, SHELLS, 6)) / (SHELLS * 6)
        b = np.random.default_rng(1).normal(size=SHELLS) * 0.1
        s, thr, modes, best = cb.time_modes(lambda t: orc.fwd_bwd(x, dy, w, b, t), repeats=steps,
                                            warm=lambda t: [orc.fwd_bwd(x, dy, w, b, t) for _ in range(warmup)])
        return _cpu_result(nvox, s, thr, modes, best, f"{nvox} voxels of the cfg4 workload per step (3 shells x 90 "
                           f"dirs, order 8, LSC 3->3 K=6), fwd + adjoint bwd, float64 port of sphdwi 0.1.0")


class Cfg2(Cfg4):
    name = "cfg2"
    metric = "voxels/s fused Signal2SH→SH2Signal round trip fwd+bwd; HBM GB/s % of peak"
    bytes_per_voxel = 4320          # x, y, dy, dx
    dom = ("rt_fwd", 2160, 0)
    # forward per tile: stage 1 3 x 6 K-steps x 3 products (128x48x16); stage 2 3 x 9 x 3 (128x96x16)
    tensor_flops_per_voxel = Cfg4.tensor_flops_per_voxel

    def __init__(self, args, dev, rank, world):
        Workload.__init__(self, args, dev, rank, world)
        import paper_1808_01517_b200 as dl

        self.shard = False
        grid = tuple(args.grid)
        self.V_subject = int(np.prod(grid))
        self.dirs, s2sh, _, sh2s = chain_modules(dev, layers=0)
        self.chain = dl.RoundTrip(s2sh, sh2s)
        assert self.chain.fused(SHELLS)
        self.params = []
        self.x, self.dy = synth_inputs(self.dirs, grid, rank, dev)
        self.x.requires_grad_(True)
        self.V_local = self.V_subject

    def _fwd(self):
        self.x.grad = None
        self.y = self.chain(self.x)

    def after_phases(self):
        pass

    def config(self):
        return {"workload": "cfg2: fused Signal2SH(order 8, 90 dirs, lambda .006) -> SH2Signal round trip fwd+bwd "
                            "(dx), one 145x174x145 subject per GPU, 3 shells x 90 dirs",
                "model": "RoundTrip", "global_batch": self.world, "voxels_per_gpu": self.V_local,
                "channels": SHELLS * NDIR, "seq_len": None, "parallelism": f"dp{self.world} (subject-sharded)",
                "l2": "no flush: each input (3.95 GB) exceeds the 126 MB L2"}

    def e2e(self):
        import torch

        dev, x, dy, chain = self.dev, self.x, self.dy, self.chain
        xh = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
        dyh = torch.empty(dy.shape, dtype=torch.float32, pin_memory=True)
        xh.copy_(x.detach())
        dyh.copy_(dy)
        res = torch.empty(1, dtype=torch.float64, pin_memory=True)
        cs = torch.cuda.Stream(device=dev)
        main = torch.cuda.current_stream(dev)
        xbuf = [torch.empty_like(x.detach()) for _ in range(2)]
        dybuf = [torch.empty_like(dy) for _ in range(2)]
        x_ready = [torch.cuda.Event() for _ in range(2)]
        dy_ready = [torch.cuda.Event() for _ in range(2)]
        freed = [torch.cuda.Event() for _ in range(2)]

        def upload(i, start=None):
            k = i % 2
            if start is not None:
                cs.wait_event(start)
            if i >= 2:
                cs.wait_event(freed[k])
            with torch.cuda.stream(cs):
                xbuf[k].copy_(xh, non_blocking=True)
                x_ready[k].record(cs)
                dybuf[k].copy_(dyh, non_blocking=True)
                dy_ready[k].record(cs)

        def e2e_step(i):
            k = i % 2
            main.wait_event(x_ready[k])
            xd = xbuf[k].detach().requires_grad_(True)
            y = chain(xd)
            main.wait_event(dy_ready[k])
            y.backward(dybuf[k])
            del y
            freed[k].record(main)
            res.copy_(xd.grad.view(-1)[:1].double(), non_blocking=True)

        upload(0)
        e2e_step(0)
        torch.cuda.synchronize()
        return _time_e2e(self, upload, e2e_step, int((xh.numel() + dyh.numel()) * 4), 8,
                         "first element of dx (float64), read back each step")

    def cpu(self, steps, warmup):
        from oracle import cpu_baseline as cb

        nvox = self.args.cpu_sample * 4
        orc = cb.ChainOracle(self.dirs)
        x, dy = cb.synthetic_sample(self.dirs, nvox)
        s, thr, modes, best = cb.time_modes(lambda t: orc.round_trip(x, dy, t), repeats=steps,
                                            warm=lambda t: [orc.round_trip(x, dy, t) for _ in range(warmup)])
        return _cpu_result(nvox, s, thr, modes, best, f"{nvox} voxels of the cfg2 workload per step (3 shells x 90 "
                           f"dirs, order 8), signal_to_sh -> sh_to_signal + adjoint, float64 port")


class Cfg5(Workload):
    name = "cfg5"
    metric = "voxels/s Signal2SH→2×LSC→SH2Signal training step (fused MSE, SGD), global batch 8 HCP subjects"
    bytes_per_voxel = 2160          # x, target
    dom = ("chain_fwd_mse", 2160 + 1080, 0)   # x, target in; dy out
    tensor_flops_per_voxel = Cfg4.tensor_flops_per_voxel
    scaling = "strong"
    GLOBAL_BATCH = 8

    def __init__(self, args, dev, rank, world):
        super().__init__(args, dev, rank, world)
        import torch

        import paper_1808_01517_b200 as dl
        from paper_1808_01517_b200.distributed import shard_range

        grid = tuple(args.grid)
        self.V_subject = int(np.prod(grid))
        self.dirs, s2sh, self.layers, sh2s = chain_modules(dev, layers=2)
        self.net = dl.SphericalChain(s2sh, self.layers, sh2s)
        self.params = [p for m in self.layers for p in m.parameters()]
        self.opt = torch.optim.SGD(self.params, lr=1e-3)
        lo, hi = shard_range(self.GLOBAL_BATCH, rank, world)
        self.subjects = list(range(lo, hi))
        self.xs = [synth_signal(self.dirs, grid, 2 * s, dev) for s in self.subjects]
        self.ts = [synth_signal(self.dirs, grid, 2 * s + 1, dev) for s in self.subjects]
        self.V_local = len(self.subjects) * self.V_subject
        self.launch_groups = len(self.subjects)

    def voxels_per_step(self):
        return self.GLOBAL_BATCH * self.V_subject

    def voxels_per_launch(self):
        return self.V_subject

    def _fwdbwd(self):
        for p in self.params:
            p.grad = None
        for x, t in zip(self.xs, self.ts):
            loss = self.net.mse_loss(x, t) * (1.0 / self.GLOBAL_BATCH)
            loss.backward()
        self.loss = loss

    def step(self):
        self._fwdbwd()
        self.after_phases()

    def phases(self):
        # the forward + backward of every local subject as one CUDA graph; the gradient all-reduce and the SGD update
        # run after it (eager: the all-reduce is a host-driven collective)
        return [("fwdbwd", self._fwdbwd)]

    def after_phases(self):
        if self.world > 1:
            from paper_1808_01517_b200.distributed import allreduce_gradients

            allreduce_gradients(self.params)
        self.opt.step()

    def config(self):
        return {"workload": "cfg5: Signal2SH(8, 90 dirs, .006) -> LSC 3->3 -> LSC 3->3 ([5], pi/5) -> SH2Signal, MSE "
                            "against a target volume (loss + dy fused into the forward kernel), backward to both "
                            "layers' weights and biases (x needs no gradient), SGD update; global batch 8 "
                            "145x174x145 subjects, 8/N per GPU",
                "model": "SphericalChain (2 LSC layers)", "global_batch": self.GLOBAL_BATCH,
                "voxels_per_gpu": self.V_local, "subjects_per_gpu": len(self.subjects), "channels": SHELLS * NDIR,
                "seq_len": None, "parallelism": f"dp{self.world} (subject-sharded, NCCL all_reduce of 114 floats)",
                "l2": "no flush: each input (3.95 GB) exceeds the 126 MB L2"}

    def e2e(self):
        """The training step from pinned host x / target buffers (H2D each step), loss read back each step."""
        import torch

        xh = torch.empty(self.xs[0].shape, dtype=torch.float32, pin_memory=True)
        th = torch.empty(self.ts[0].shape, dtype=torch.float32, pin_memory=True)
        xh.copy_(self.xs[0])
        th.copy_(self.ts[0])
        lh = torch.empty(1, dtype=torch.float32, pin_memory=True)
        xd, td = torch.empty_like(self.xs[0]), torch.empty_like(self.ts[0])

        def upload(i, start=None):
            pass

        def e2e_step(i):
            self.opt.zero_grad(set_to_none=True)
            for _ in self.subjects:
                xd.copy_(xh, non_blocking=True)
                td.copy_(th, non_blocking=True)
                loss = self.net.mse_loss(xd, td) * (1.0 / self.GLOBAL_BATCH)
                loss.backward()
            if self.world > 1:
                from paper_1808_01517_b200.distributed import allreduce_gradients

                allreduce_gradients(self.params)
            self.opt.step()
            lh.copy_(loss.detach().view(1), non_blocking=True)

        e2e_step(0)
        torch.cuda.synchronize()
        n_sub = len(self.subjects)
        return _time_e2e(self, upload, e2e_step, int((xh.numel() + th.numel()) * 4 * n_sub), 4, "the step's loss",
                         pipeline="x and target uploaded synchronously before each subject's pass")

    def cpu(self, steps, warmup):
        from oracle import cpu_baseline as cb

        nvox = self.args.cpu_sample
        orc = cb.ChainOracle(self.dirs)
        x, t = cb.synthetic_sample(self.dirs, nvox)
        layers = [(np.random.default_rng(1 + k).normal(size=(3, 3, 6)) / 18, np.random.default_rng(1 + k).normal(size=3) * 0.1)
                  for k in range(2)]
        s, thr, modes, best = cb.time_modes(lambda th: orc.train_step(x, t, layers, th), repeats=steps,
                                            warm=lambda th: [orc.train_step(x, t, layers, th) for _ in range(warmup)])
        return _cpu_result(nvox, s, thr, modes, best, f"{nvox} voxels of one cfg5 subject per step (2 LSC layers, "
                           f"MSE, backward to both layers), float64 port")


class Cfg1(Workload):
    name = "cfg1"
    metric = "voxels/s Signal2SH forward (order 8, 90 dirs, 1 shell); HBM GB/s % of peak"
    dtype = "f32 (SIMT fp32 FMA)"
    bytes_per_voxel = 540           # x in (90), c out (45)
    dom = ("chan_contract", 540, None)
    flush_l2 = True

    def __init__(self, args, dev, rank, world):
        super().__init__(args, dev, rank, world)
        import paper_1808_01517_b200 as dl
        from paper_1808_01517_b200.directions import unit_sphere_directions

        self.dirs = unit_sphere_directions(NDIR)
        self.s2sh = dl.Signal2SH(ORDER, self.dirs, lb_lambda=LAM).to(dev)
        self.x = synth_signal(self.dirs, (32, 32, 32), rank, dev, shells=1)
        self.V_local = 32 ** 3

    def voxels_per_step(self):
        return self.world * self.V_local

    def step(self):
        self.c = self.s2sh(self.x)

    def config(self):
        return {"workload": "cfg1: Signal2SH(order 8, 90 dirs, lambda .006) forward, one 32^3 subject per GPU",
                "model": "Signal2SH", "global_batch": self.world, "voxels_per_gpu": self.V_local, "channels": NDIR,
                "seq_len": None, "parallelism": f"replicas x{self.world}",
                "l2": "flushed between timed steps (256 MB write)"}

    def e2e(self):
        import torch

        xh = torch.empty(self.x.shape, dtype=torch.float32, pin_memory=True)
        xh.copy_(self.x)
        ch = torch.empty((1, 45, 32, 32, 32), dtype=torch.float32, pin_memory=True)

        def e2e_step(i):
            c = self.s2sh(xh.to(self.dev, non_blocking=True))
            ch.copy_(c, non_blocking=True)

        e2e_step(0)
        torch.cuda.synchronize()
        return _time_e2e(self, lambda i, start=None: None, e2e_step, xh.numel() * 4, ch.numel() * 4,
                         "the SH coefficients c (whole output)", pipeline="synchronous H2D, compute, D2H")

    def cpu(self, steps, warmup):
        from oracle import cpu_baseline as cb

        nvox = 32 ** 3
        orc = cb.ChainOracle(self.dirs, shells=1)
        x, _ = cb.synthetic_sample(self.dirs, nvox, shells=1)
        s, thr, modes, best = cb.time_modes(lambda t: orc.signal_to_sh(x, t), repeats=max(steps, 5),
                                            warm=lambda t: [orc.signal_to_sh(x, t) for _ in range(warmup)])
        return _cpu_result(nvox, s, thr, modes, best, "the whole cfg1 volume (32^3 voxels x 90 dirs), float64 port")


class Cfg3(Workload):
    name = "cfg3"
    metric = "voxels/s LocalSphericalConvolution 1->1 fwd+bwd (order 8, 90 origins, [5] ring); HBM GB/s % of peak"
    dtype = "f32 (SIMT fp32 FMA; float64 Gram finalize)"
    bytes_per_voxel = 900           # c_in, c_out, g, c_in, dc_in
    dom = ("lsc_fwd", 360, None)
    flush_l2 = True

    def __init__(self, args, dev, rank, world):
        super().__init__(args, dev, rank, world)
        import torch

        import paper_1808_01517_b200 as dl
        from paper_1808_01517_b200.directions import unit_sphere_directions

        self.dirs = unit_sphere_directions(NDIR)
        self.lsc = dl.LocalSphericalConvolution(1, 1, ORDER, ORDER, self.dirs, [5], lb_lambda=LAM,
                                                angular_distance=math.pi / 5).to(dev)
        self.lsc.load_kernel(dl.LscKernel(np.random.default_rng(3).normal(size=(1, 1, 6)) / 6,
                                          np.random.default_rng(3).normal(size=1) * 0.1))
        gen = torch.Generator(device=dev).manual_seed(rank)
        self.c_in = (torch.rand((4, 45, 32, 32, 32), generator=gen, device=dev) - 0.5).requires_grad_(True)
        self.g = torch.randn((4, 45, 32, 32, 32), generator=gen, device=dev)
        self.params = list(self.lsc.parameters())
        self.V_local = 4 * 32 ** 3

    def voxels_per_step(self):
        return self.world * self.V_local

    def _fwd(self):
        self.c_in.grad = None
        for p in self.params:
            p.grad = None
        self.u = self.lsc(self.c_in)

    def _bwd(self):
        self.u.backward(self.g)

    def step(self):
        self._fwd()
        self._bwd()

    def phases(self):
        return [("fwd", self._fwd), ("bwd", self._bwd)]

    def config(self):
        return {"workload": "cfg3: LocalSphericalConvolution 1->1 (order 8, 90 origins, [5] ring at pi/5, lambda "
                            ".006) fwd+bwd (dc, dW, db) on a batch of 4 32^3 SH patches per GPU",
                "model": "LocalSphericalConvolution", "global_batch": 4 * self.world, "voxels_per_gpu": self.V_local,
                "channels": 45, "seq_len": None, "parallelism": f"replicas x{self.world}",
                "l2": "flushed between timed steps (256 MB write)"}

    def e2e(self):
        import torch

        ch = torch.empty(self.c_in.shape, dtype=torch.float32, pin_memory=True)
        gh = torch.empty(self.g.shape, dtype=torch.float32, pin_memory=True)
        ch.copy_(self.c_in.detach())
        gh.copy_(self.g)
        wh = torch.empty(self.lsc.sconv.weight.shape, pin_memory=True)
        bh = torch.empty(self.lsc.sconv.bias.shape, pin_memory=True)

        def e2e_step(i):
            for p in self.params:
                p.grad = None
            c = ch.to(self.dev, non_blocking=True).requires_grad_(True)
            u = self.lsc(c)
            u.backward(gh.to(self.dev, non_blocking=True))
            wh.copy_(self.lsc.sconv.weight.grad, non_blocking=True)
            bh.copy_(self.lsc.sconv.bias.grad, non_blocking=True)

        e2e_step(0)
        torch.cuda.synchronize()
        return _time_e2e(self, lambda i, start=None: None, e2e_step, (ch.numel() + gh.numel()) * 4,
                         (wh.numel() + bh.numel()) * 4, "LSC dW, db", pipeline="synchronous H2D, compute, D2H")

    def cpu(self, steps, warmup):
        from oracle import cpu_baseline as cb

        nvox = 32 ** 3
        orc = cb.ChainOracle(self.dirs, shells=1)
        rng = np.random.default_rng(3)
        c = rng.uniform(-0.5, 0.5, size=(1, 45, nvox))
        g = rng.normal(size=(1, 45, nvox))
        w = rng.normal(size=(1, 1, 6)) / 6
        b = rng.normal(size=1) * 0.1
        s, thr, modes, best = cb.time_modes(lambda t: orc.lsc_fwd_bwd(c, g, w, b, t), repeats=max(steps, 3),
                                            warm=lambda t: [orc.lsc_fwd_bwd(c, g, w, b, t) for _ in range(warmup)])
        return _cpu_result(nvox, s, thr, modes, best, "one of the 4 cfg3 patches per step (32^3 voxels), LSC fwd + "
                           "adjoint, float64 port")


def _cpu_result(nvox, sec, threads, modes, best, sample):
    return {"value": nvox / sec, "sec": sec, "cores": threads, "modes": modes, "best": best, "sample": sample}


WORKLOADS = {"cfg1": Cfg1, "cfg2": Cfg2, "cfg3": Cfg3, "cfg4": Cfg4, "cfg5": Cfg5}


def _time_e2e(w, upload, e2e_step, h2d, d2h, result, pipeline="inputs uploaded on a copy stream into two buffer "
              "sets, overlapping the previous step's compute"):
    import torch
    import torch.distributed as dist

    from paper_1808_01517_b200.distributed import max_over_ranks

    if w.world > 1:
        dist.barrier()
    n = max(2, min(w.args.steps, 5))
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    upload(0, start=s0)
    upload(1, start=s0)
    for i in range(n):
        e2e_step(i)
        if i + 2 < n:
            upload(i + 2)
    s1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(s0.elapsed_time(s1) / n, w.dev)
    return {"value": w.voxels_per_step() / (ms / 1e3), "unit": "voxels/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": ms, "steps": n, "result_read": result,
            "pipeline": pipeline}


# ----------------------------------------------------------------------------- CPU reference arm
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    w = WORKLOADS[args.config]
    import torch  # noqa: F401  (same import cost as our arm)

    from paper_1808_01517_b200.directions import unit_sphere_directions

    stub = w.__new__(w)
    stub.args, stub.dirs = args, unit_sphere_directions(NDIR)
    r = stub.cpu(args.steps, args.warmup)
    value = r["value"]
    line = {
        "impl": "reference", "metric": w.metric, "value": value, "unit": "voxels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["sec"] * 1e3, "higher_is_better": True,
        "scaling": w.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} (bounded voxel sample per step, float64 CPU port)",
                   "parallelism": "cpu, best of: " + ", ".join(f"{k} {v * 1e3:.1f} ms" for k, v in r["modes"].items())},
        "cpu_baseline": {"value": value, "unit": "voxels/s", "cores": r["cores"], "kind": "port",
                         "sample": f"{r['sample']}; threading mode {r['best']} (the faster of the reference's two "
                                   f"modes)"},
        "e2e": {"value": value, "unit": "voxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1808_01517_b200 import _lib
    from paper_1808_01517_b200.distributed import max_over_ranks

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() < 1:
        raise SystemExit("bench.py: no CUDA device")
    # --dist-backend gloo (a test mode): ranks may share GPUs (local rank modulo the visible devices); the kernels of
    # different ranks never wait on one another -- the only exchange is the host-side all-reduce
    dev = torch.device("cuda", local % torch.cuda.device_count() if args.dist_backend == "gloo" else local)
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    W = WORKLOADS[args.config](args, dev, rank, world)
    graphed = W.graphed and not args.no_graph
    flush = _l2_flush_buffer(dev) if W.flush_l2 else None

    for _ in range(args.warmup):
        W.step()
    torch.cuda.synchronize()
    W.drop()

    graphs, graph_launches = [], 0
    _lib.ktimer_arm(True)   # eager: events around each fused-kernel launch; graphed: armed for the capture below
    if graphed:
        # Replay the step as CUDA graphs (one per phase): the same kernels and buffers without the host launches
        # and the Python / autograd work between them.  The kernel timer is armed during capture, so the fused
        # kernels' launches are bracketed by external event nodes that every replay re-records: after the timed
        # loop they hold the durations of the kernels inside the LAST timed step.
        pool = torch.cuda.graph_pool_handle()
        c0 = _lib.total_launches()
        for name, fn in W.phases():
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=pool):
                fn()
            graphs.append((name, g))
        torch.cuda.synchronize()
        graph_launches = _lib.total_launches() - c0

    phase_ev = []

    phase_names = [name for name, _ in graphs] if graphed else ["step"]

    def step(record):
        if flush is not None:
            flush.zero_()   # before the step's first event: the flush is not timed
        evs = []

        def mark():
            if record:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                evs.append(e)

        if graphed:
            for _, g in graphs:
                mark()
                g.replay()
        else:
            mark()
            W.step()
        mark()
        if record:
            phase_ev.append(evs)
        if graphed:
            W.after_phases()

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    uuid = None
    try:
        uuid = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        pass
    clocks = ClockSampler(uuid) if (rank == 0 and not args.no_clocks) else None
    if clocks:
        clocks.start()
    if not args.no_clocks:   # every rank (the steps hold collectives): keep the GPU loaded while the sampler spins up
        for _ in range(max(1, args.warmup)):
            step(False)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = _lib.total_launches()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(args.steps):
        step(True)
    end.record()
    torch.cuda.synchronize()
    launches = graph_launches * args.steps if graphed else _lib.total_launches() - n0
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    if flush is not None:   # L2 flushed before every step: the step is timed from its first to its last event
        ms = statistics.mean(ev[0].elapsed_time(ev[-1]) for ev in phase_ev)
    else:
        ms = start.elapsed_time(end) / args.steps
    ms = max_over_ranks(ms, dev)
    phase_ms = {}
    for i, name in enumerate(phase_names):
        phase_ms[name] = statistics.mean(ev[i].elapsed_time(ev[i + 1]) for ev in phase_ev)

    # Dominant-kernel durations inside the timed steps: the library's kernel timer stamps %globaltimer when a
    # launch's first CTA starts and its last CTA ends (device-side, so it works inside the replayed graphs and
    # times the kernel alone); every timed step's launches are in the ring -- mean over them, reconciled with
    # the step time.
    kern = None
    nl = min(args.steps * W.launch_groups, 60)   # the ring holds the last 63 launches per slot
    if W.dom and W.dom[2] is not None:
        try:
            def med(slot):   # mean over the timed launches (comparable with the mean phase times), then min, max
                if _lib.ktimer_count(slot) < nl:
                    return None
                v = [_lib.ktimer_read(slot, b) for b in range(nl)]
                return statistics.mean(v), min(v), max(v)

            f, b_, g_ = med(0), med(1), med(2)
            if f:
                kern = {"fwd_ms": f[0], "fwd_min_max": f[1:],
                        "how": f"mean over the {nl} launches of the timed steps: device %globaltimer stamps at the "
                               f"kernel's first CTA start and last CTA end (inside the replayed graph)" if graphed else
                               f"mean over the {nl} launches of the timed steps: device %globaltimer stamps at the "
                               f"kernel's first CTA start and last CTA end"}
                if b_:
                    kern["bwd_ms"], kern["bwd_min_max"] = b_[0], b_[1:]
                if g_:
                    kern["gram_ms"], kern["gram_min_max"] = g_[0], g_[1:]
        except Exception as exc:
            log(f"kernel timer unavailable ({exc})")
            kern = None
    _lib.ktimer_arm(False)
    recon = None
    if kern:
        ksum = (kern["fwd_ms"] + kern.get("bwd_ms", 0.0) + kern.get("gram_ms", 0.0)) * W.launch_groups
        fwd_phase = phase_ms.get("fwd", phase_ms.get("step", ms))
        recon = {"kernels_ms": ksum, "ms_per_step": ms, "share": ksum / ms, "launch_groups": W.launch_groups,
                 "fwd_kernel_le_phase": kern["fwd_ms"] * (1 if "fwd" in phase_ms else W.launch_groups) <= fwd_phase * 1.0005,
                 "ok": ksum <= ms * 1.0005}
        if not recon["ok"] or not recon["fwd_kernel_le_phase"]:
            log(f"kernel timer does not reconcile with the step ({recon}); roofline falls back to the phase time")
            kern["rejected"] = True

    # free the graphs (and the autograd state they keep alive) before the e2e leg
    graphs.clear()
    W.drop()
    torch.cuda.synchronize()
    e2e = None if args.no_e2e else W.e2e()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r = W.cpu(3, 1)
        cpu = {"value": r["value"], "unit": "voxels/s", "cores": r["cores"], "kind": "port",
               "sample": f"{r['sample']}; median of 3 after 1 warm-up, faster threading mode {r['best']} (" +
                         ", ".join(f"{k} {v * 1e3:.1f} ms" for k, v in r["modes"].items()) + ")"}

    if rank == 0:
        peak, peak_tf, peak_kind = measured_peaks()
        V_local = W.voxels_per_launch()
        dname, dbytes_vox, slot = W.dom
        launch_ms, how = None, None
        if kern and not kern.get("rejected"):
            launch_ms, how = kern["fwd_ms"], "kernel launches inside the timed steps (device timestamps, mean)"
        else:
            launch_ms = phase_ms.get("fwd", phase_ms.get("step", ms))
            how = "the whole forward phase of the timed step (graph replay; includes small operator kernels)"
        nbytes = dbytes_vox * V_local
        achieved = nbytes / (launch_ms / 1e3) / 1e9
        traffic = ncu_traffic(dname)
        roof = {"bound": "hbm", "kernel": dname, "timing": how, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_kind": peak_kind, "frac_of_8tbs": achieved / NOMINAL_HBM,
                "algorithmic_bytes_per_launch": nbytes, "bytes_per_voxel_per_launch": dbytes_vox,
                "launch_ms": launch_ms, "traffic": traffic,
                "traffic_ratio": (traffic / nbytes) if traffic else None}
        if W.tensor_flops_per_voxel:
            tflops = W.tensor_flops_per_voxel * V_local / (launch_ms / 1e3) / 1e12
            roof["tensor"] = {"flops_per_launch": W.tensor_flops_per_voxel * V_local, "achieved_tflops": tflops,
                              "peak_tflops": peak_tf, "frac": tflops / peak_tf,
                              "pipe_active_pct_ncu": ncu_traffic(dname, "tensor_pipe_active_pct"),
                              "note": "MMA flops the kernel issues (fp16 split-term products) over its duration, "
                                      "against the measured dense bf16 GEMM rate; pipe_active_pct_ncu: "
                                      "sm__pipe_tensor_cycles_active from the committed ncu capture"}
        step_bytes = W.bytes_per_voxel * W.voxels_per_step() / max(world, 1)
        line = {
            "metric": W.metric, "value": W.voxels_per_step() / (ms / 1e3), "unit": "voxels/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": W.scaling, "vs_baseline": None, "dtype": W.dtype, "data": "synthetic",
            "config": dict(W.config(), cuda_graph=graphed),
            "roofline": roof,
            "step_hbm": {"bytes_per_voxel": W.bytes_per_voxel, "gbs": step_bytes / (ms / 1e3) / 1e9,
                         "frac": step_bytes / (ms / 1e3) / 1e9 / peak,
                         "frac_of_8tbs": step_bytes / (ms / 1e3) / 1e9 / NOMINAL_HBM},
            "phase_ms": phase_ms or None,
            "kernel_ms": kern,
            "reconcile": recon,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="cfg4")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--shard", choices=["subjects", "voxels"], default="subjects",
                    help="cfg4 at N > 1: a subject per rank (weak) or one subject in X-slabs (strong)")
    ap.add_argument("--grid", type=int, nargs=3, default=list(GRID))
    ap.add_argument("--cpu-sample", type=int, default=65536, help="voxels per CPU-reference step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time the eager autograd step instead of CUDA graphs")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: test mode in which ranks may share a GPU (multi-rank logic on a 1-GPU box)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: fewer than 3 warm-up steps")
    if args.impl == "reference":
        run_reference(args)
        return
    maybe_spawn(args)
    run_ours(args)


if __name__ == "__main__":
    main()
