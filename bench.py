#!/usr/bin/env python
"""Benchmark: fused Signal2SH -> LSC -> SH2Signal forward + backward on HCP-sized volumes.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun (one rank per GPU, NCCL); every rank processes its own
HCP-sized subject (weak scaling, subject sharding) and the LSC parameter gradients are
summed with one bucketed NCCL all_reduce per step.  Rank 0 prints ONE JSON line.

Workload (BASELINE.json configs[3]): x = (1, 3*90, 145, 174, 145) fp32 per GPU, synthetic
band-limited signals (phantom.py:77-88 distribution) + N(0, 0.02^2) noise; upstream grad
dy ~ N(0, 1); Signal2SH(8, 90 dirs, lambda=0.006) -> LSC 3->3 ([5] ring, pi/5, lambda=0.006)
-> SH2Signal(8, 90 dirs).  Inputs (3.95 GB each) exceed the 126 MB L2, so no flush is needed.
"""

from __future__ import annotations

import argparse
import json
import math
import os
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
FALLBACK_HBM = 6650.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def ncu_traffic(kernel: str):
    """Per-launch dram bytes for `kernel` from the committed ncu summary, else None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

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
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- model / inputs
def build_model(dev):
    import paper_1808_01517_b200 as dl
    from paper_1808_01517_b200.directions import unit_sphere_directions

    dirs = unit_sphere_directions(NDIR)
    s2sh = dl.Signal2SH(ORDER, dirs, lb_lambda=LAM).to(dev)
    lsc = dl.LocalSphericalConvolution(SHELLS, SHELLS, ORDER, ORDER, dirs, [5], lb_lambda=LAM,
                                       angular_distance=math.pi / 5).to(dev)
    w = np.random.default_rng(1).normal(size=(SHELLS, SHELLS, 6)) / (SHELLS * 6)
    b = np.random.default_rng(1).normal(size=SHELLS) * 0.1
    lsc.load_kernel(dl.LscKernel(w, b))
    sh2s = dl.SH2Signal(ORDER, dirs).to(dev)
    return dirs, lsc, dl.SphericalChain(s2sh, lsc, sh2s)


def synth_inputs(dirs, grid, seed, dev):
    """Band-limited synthetic DWI (phantom.py:77-88 distribution) + noise, generated on the device."""
    import torch

    from paper_1808_01517_b200.geometry import basis_degrees, eval_basis

    V = int(np.prod(grid))
    B = torch.tensor(eval_basis(dirs, ORDER), dtype=torch.float32, device=dev)
    l = torch.tensor(basis_degrees(ORDER), dtype=torch.float32, device=dev)
    amp = 0.9 / (1.0 + l * (l + 1.0) / 4.0)
    x = torch.empty((1, SHELLS * NDIR, V), dtype=torch.float32, device=dev)
    for s in range(SHELLS):
        g = torch.Generator(device=dev).manual_seed(1000 + s + 7919 * seed)
        coeffs = (torch.rand((B.shape[1], V), generator=g, device=dev) * 2 - 1) * amp[:, None]
        coeffs[0] = 2.0 * math.sqrt(math.pi)
        x[0, s * NDIR:(s + 1) * NDIR] = B @ coeffs
        x[0, s * NDIR:(s + 1) * NDIR] += 0.02 * torch.randn((NDIR, V), generator=g, device=dev)
        del coeffs
    g = torch.Generator(device=dev).manual_seed(2 + 7919 * seed)
    dy = torch.randn((1, SHELLS * NDIR, V), generator=g, device=dev)
    return x.view(1, SHELLS * NDIR, *grid), dy.view(1, SHELLS * NDIR, *grid)


# ----------------------------------------------------------------------------- CPU reference arm
def cpu_reference(nvox: int, steps: int, warmup: int):
    from oracle import cpu_baseline as cb
    from paper_1808_01517_b200.directions import unit_sphere_directions

    dirs = unit_sphere_directions(NDIR)
    orc = cb.ChainOracle(dirs)
    x, dy = cb.synthetic_sample(dirs, nvox)
    w = np.random.default_rng(1).normal(size=(SHELLS, SHELLS, 6)) / (SHELLS * 6)
    b = np.random.default_rng(1).normal(size=SHELLS) * 0.1
    cores = cb.host_cores()
    for _ in range(warmup):
        orc.fwd_bwd(x, dy, w, b, cores)
    t0 = time.perf_counter()
    for _ in range(steps):
        orc.fwd_bwd(x, dy, w, b, cores)
    dt = time.perf_counter() - t0
    return steps * nvox / dt, dt / steps, cores


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    nvox = args.cpu_sample
    value, sec, cores = cpu_reference(nvox, args.steps, args.warmup)
    sample = (f"{nvox} voxels/step of the cfg4 workload (3 shells x 90 dirs, order 8, LSC 3->3 K=6), float64 "
              f"oracle port of sphdwi 0.1.0 forward + per-stage adjoint backward, threads={cores}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "voxels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg4 fused Signal2SH->LSC->SH2Signal fwd+bwd (bounded voxel sample per step)",
                   "voxels_per_step": nvox, "parallelism": f"cpu threads={cores}"},
        "cpu_baseline": {"value": value, "unit": "voxels/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "voxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1808_01517_b200 import _lib
    from paper_1808_01517_b200.distributed import allreduce_gradients, max_over_ranks

    world, rank, local = dist_env()
    assert world == args.gpus or world == 1, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    grid = tuple(args.grid)
    V = int(np.prod(grid))
    dirs, lsc, chain = build_model(dev)
    x, dy = synth_inputs(dirs, grid, rank, dev)
    x.requires_grad_(True)
    params = list(lsc.parameters())

    fwd_ev, bwd_ev = [], []

    def step(record):
        x.grad = None
        for p in params:
            p.grad = None
        if record:
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
        y = chain(x)
        if record:
            e1.record()
        y.backward(dy)
        if record:
            e2.record()
            fwd_ev.append((e0, e1))
            bwd_ev.append((e1, e2))
        if world > 1:
            allreduce_gradients(params)
        return y

    eager_step = step
    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if not args.no_graph:
        # Replay the step as two CUDA graphs (forward, backward): the same kernels and buffers, without
        # ~20 host launches and the Python/autograd work between them.  Gradients are written (not
        # accumulated) on every replay, exactly like the eager step with .grad reset to None.
        x.grad = None
        for p in params:
            p.grad = None
        pool = torch.cuda.graph_pool_handle()
        g_fwd, g_bwd = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        c0 = _lib.total_launches()
        with torch.cuda.graph(g_fwd, pool=pool):
            y_static = chain(x)
        with torch.cuda.graph(g_bwd, pool=pool):
            y_static.backward(dy)
        torch.cuda.synchronize()
        graph_launches = _lib.total_launches() - c0   # our kernels captured per step

        def step(record):  # noqa: F811 -- graphed replacement of the eager step above
            if record:
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record()
            g_fwd.replay()
            if record:
                e1.record()
            g_bwd.replay()
            if record:
                e2.record()
                fwd_ev.append((e0, e1))
                bwd_ev.append((e1, e2))
            if world > 1:
                allreduce_gradients(params)
            return y_static

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
        for _ in range(max(1, args.warmup)):     # keep the GPU loaded while the sampler spins up
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
    launches = _lib.total_launches() - n0
    if not args.no_graph:
        launches = graph_launches * args.steps   # replays do not pass through the host launch counter
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    ms = start.elapsed_time(end) / args.steps
    ms = max_over_ranks(ms, dev)
    fwd_ms = statistics.mean(a.elapsed_time(b) for a, b in fwd_ev)
    bwd_ms = statistics.mean(a.elapsed_time(b) for a, b in bwd_ev)
    # The dominant kernel's own launch duration: CUDA events that dl_ktimer_* records on the kernel's stream
    # around each fused-chain launch, over K eager steps run right after the timed region (same kernels, inputs
    # and buffers), each read once the stream has passed it.  Measured alternatives, both noisier: event nodes
    # captured inside the graphs read longer than the whole forward phase, and eager steps run back to back
    # without the per-step synchronize spread 2.0-2.7 ms per launch.
    kern = None
    try:
        _lib.ktimer_arm(True)
        kf, kb = [], []
        for _ in range(args.steps):
            eager_step(False)
            torch.cuda.synchronize()
            kf.append(_lib.ktimer_read(0))
            kb.append(_lib.ktimer_read(1))
        kern = {"fwd_ms": statistics.median(kf), "bwd_ms": statistics.median(kb), "samples": len(kf),
                "fwd_ms_min_max": [min(kf), max(kf)], "bwd_ms_min_max": [min(kb), max(kb)],
                "how": "median of CUDA events around the chain2h_tc launch on its stream, one eager step at a time "
                       "after the timed region"}
    except Exception as exc:   # a non-default kernel selection (no fp16 chain2h pass): fall back to the phase
        log(f"kernel timer unavailable ({exc}); roofline uses the forward phase time")
    finally:
        _lib.ktimer_arm(False)

    # ---- end to end through the public API with host buffers (pinned), same metric ----
    e2e = None
    if not args.no_e2e:
        xh = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
        dyh = torch.empty(dy.shape, dtype=torch.float32, pin_memory=True)
        xh.copy_(x.detach())
        dyh.copy_(dy)
        wh = torch.empty(lsc.sconv.weight.shape, pin_memory=True)
        bh = torch.empty(lsc.sconv.bias.shape, pin_memory=True)

        # Input pipeline: a copy stream uploads step i's x and dy into one of two device buffer sets while the
        # compute stream runs step i - 1 (x first, so the forward starts before dy has arrived).  Every step's
        # inputs still cross PCIe inside the timed region; only their overlap with compute is new.
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
                cs.wait_event(freed[k])   # step i - 2 is done with this buffer set
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
            freed[k].record(main)
            if world > 1:
                allreduce_gradients(params)
            wh.copy_(lsc.sconv.weight.grad, non_blocking=True)
            bh.copy_(lsc.sconv.bias.grad, non_blocking=True)

        upload(0)
        e2e_step(0)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        n_e2e = max(2, min(args.steps, 5))
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        upload(0, start=s0)
        upload(1, start=s0)
        for i in range(n_e2e):
            e2e_step(i)
            if i + 2 < n_e2e:
                upload(i + 2)
        s1.record()
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(s0.elapsed_time(s1) / n_e2e, dev)
        e2e = {"value": world * V / (e2e_ms / 1e3), "unit": "voxels/s",
               "h2d_bytes_per_step": int((xh.numel() + dyh.numel()) * 4),
               "d2h_bytes_per_step": int((wh.numel() + bh.numel()) * 4), "ms_per_step": e2e_ms,
               "steps": n_e2e, "result_read": "LSC dW, db (the step's parameter gradients)",
               "pipeline": "inputs uploaded on a copy stream into two buffer sets, overlapping compute"}
        del xh, dyh, xbuf, dybuf

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        value, sec, cores = cpu_reference(args.cpu_sample, 3, 1)
        cpu = {"value": value, "unit": "voxels/s", "cores": cores, "kind": "port",
               "sample": f"{args.cpu_sample} voxels of the same workload, fwd+bwd, 3 timed reps after 1 warm-up "
                         f"(float64 oracle port of sphdwi 0.1.0 + adjoint restatement, {cores} threads)"}

    if rank == 0:
        peak, peak_kind = measured_peak_hbm()
        fwd_bytes = V * (SHELLS * NDIR + SHELLS * NDIR) * 4            # x in, y out
        bwd_bytes = V * (3 * SHELLS * NDIR) * 4                        # dy in, x-or-c in, dx out
        # dominant kernel: the fused chain kernel (forward and adjoint launches take the same time; the
        # forward phase is one fp16-pass launch, the ~7 us bf16 check pass and ~25 us of operator folding /
        # packing).  Algorithmic bytes of one launch: x in + y out (SURVEY.md 8(d), 2,160 B/voxel at cfg4).
        dom = ("chain_fwd", fwd_bytes, kern["fwd_ms"] if kern else fwd_ms)
        if kern:
            kname = "chain2h_tc fp16 pass, forward (kernel launch, CUDA events on its stream)"
        elif "DELIMIT_SPLIT_TERMS" in os.environ:
            kname = "chain3v_tc bf16 (forward phase)"
        elif "DELIMIT_NO_CHAIN2H" in os.environ:
            kname = "chain3v_tc fp16 pass + bf16 check (forward phase)"
        else:
            kname = "chain2h_tc fp16 pass + bf16 check (forward phase)"
        achieved = dom[1] / (dom[2] / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": world * V / (ms / 1e3), "unit": "voxels/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "cfg4: fused Signal2SH(order 8, 90 dirs, lambda .006) -> LSC 3->3 ([5] ring, "
                                   "pi/5) -> SH2Signal fwd+bwd, one 145x174x145 subject per GPU",
                       "model": "SphericalChain", "global_batch": world, "voxels_per_gpu": V,
                       "channels": SHELLS * NDIR, "seq_len": None, "parallelism": f"dp{world} (subject-sharded)",
                       "l2": "no flush: each input (3.95 GB) exceeds the 126 MB L2",
                       "cuda_graph": not args.no_graph},
            "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                         "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": dom[1], "launch_ms": dom[2],
                         "bytes_per_voxel": 2160, "traffic": ncu_traffic(dom[0]),
                         # DRAM bytes the launch actually moves (algorithmic x + y plus the Gram term planes,
                         # profiles/ncu_traffic.json) over the same time: how close the memory system runs
                         "dram_gbs": (ncu_traffic(dom[0]) or 0) / (dom[2] / 1e3) / 1e9 or None,
                         "dram_frac": ((ncu_traffic(dom[0]) or 0) / (dom[2] / 1e3) / 1e9) / peak or None},
            "phase_ms": {"fwd": fwd_ms, "bwd": bwd_ms},
            "kernel_ms": kern,
            # the same algorithmic bytes over the whole forward phase (operator folding / packing, the chain
            # kernel and the bf16 check pass)
            "fwd_phase_hbm_frac": fwd_bytes / (fwd_ms / 1e3) / 1e9 / peak,
            "step_hbm_gbs": (fwd_bytes + bwd_bytes) / (ms / 1e3) / 1e9,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--grid", type=int, nargs=3, default=list(GRID))
    ap.add_argument("--cpu-sample", type=int, default=65536, help="voxels per CPU-reference step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time the eager autograd step instead of its CUDA graphs")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: fewer than 3 warm-up steps")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
