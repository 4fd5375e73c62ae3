#!/usr/bin/env python3
"""bench.py -- S4ConvD depthwise conv1d fwd + dX + dW step on B200.

Metric (BASELINE.json): effective HBM GB/s and % of the HBM roofline per path
(fwd / dX / dW), and fwd+bwd conv time per step.

* A "step" is one pass of the hot path over one batch: y = forward(x,k), then
  the layer's backward dx = backward_input(gy,k), dk = backward_weight(gy,x)
  (+ the dW combine over ranks when N > 1), all through the library's C ABI
  on resident device buffers.  Inputs come from the reference's splitmix64
  stream generated in place on the device.
* Default workload: BASELINE config 3 (B=256, H=512, L=8192, K=7, fp32), the
  largest single-GPU config and the one the north star's roofline targets are
  stated on.  4 GiB per tensor >> 126 MB L2, so no L2 flush is needed.
  Default multiply-add mode: Separate, the reference's default
  (conv_core.hpp:50,57) -- both arms compute bit-identical y / dX.
* value = the step's compulsory HBM bytes over all ranks / device step time
  (CUDA events, max over ranks).  Compulsory bytes of one step: forward reads
  x and k and writes y; the backward reads gy, x and k and writes dx and dk:
  20*B*H*L + 12*H*K.  (The per-path table keeps the reference's per-path
  logical bytes, 8*B*H*L + 4*H*K each, src/exec_model.cpp:168-179.)  The
  reference arm divides the same bytes by its own time, so the two values'
  ratio is the time ratio.
* Scaling: weak by default (every rank runs the config's batch, global batch
  B*N); --global-batch G fixes the global batch and shards it with
  ks_shard_rows (strong scaling, BASELINE configs 4 and 5).
* e2e: the same metric end to end from pinned host memory, H2D/D2H inside the
  timed region, through the drop-in's three host calls (forward,
  backward_input, backward_weight: the reference's value-type API); the
  library's one-call ks_dwconv1d_step_f32_host is reported beside it.
* --impl reference: the reference's own CPU conv_core.cpp (oracle/_ref, built
  from /root/reference) on the host cores, channel-sliced over threads, on a
  bounded channel sample of the same workload, in the same mode.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {  # BASELINE.json configs, name -> (B, H, L, K)
    "config1": (16, 64, 1024, 64),
    "config2": (64, 128, 4096, 4096),
    "config3": (256, 512, 8192, 7),
    "config4": (1024, 256, 2048, 256),
    "config5a": (512, 1024, 16384, 16),
    "config5b": (512, 1024, 16384, 128),
    "config5c": (512, 1024, 16384, 1024),
}
WORKLOAD = {
    "config1": "reference fixture depthwise conv1d fwd+dX+dW fp32 (16,64,1024,64)",
    "config2": "S4ConvD training-shape layer fp32 (64,128,4096,K=L=4096) fwd+bwd",
    "config3": "short-kernel depthwise conv1d fwd+dX+dW fp32 (256,512,8192,7), bandwidth-bound",
    "config4": "dW-dominated reduction case fp32 (1024,256,2048,256)",
    "config5a": "S4ConvD stack sweep fp32 (512,1024,16384,16)",
    "config5b": "S4ConvD stack sweep fp32 (512,1024,16384,128)",
    "config5c": "S4ConvD stack sweep fp32 (512,1024,16384,1024)",
}
METRIC = "effective HBM GB/s & % roofline per path (fwd/dX/dW); fwd+bwd conv time/step"


def path_bytes(B, H, L, K):
    """Algorithmic bytes per path: read one [B,H,L] tensor + k, write one
    [B,H,L] tensor (fwd: x,k->y; dX: gy,k->dx; dW: gy,x->dk)."""
    return 8 * B * H * L + 4 * H * K


def step_bytes(B, H, L, K):
    """Compulsory HBM bytes of one training step of the layer: forward reads x,
    k and writes y; the backward reads gy, x, k and writes dx, dk."""
    return 20 * B * H * L + 12 * H * K


def path_flops(B, H, L, K):
    return 2 * B * H * L * K  # reference src/analyzer.cpp:36-49


def useful_flops(B, H, L, K):
    """2 x the taps that touch the row: the paper's count includes
    taps on the zero padding, 25% of them at K = L.  Same total for fwd (sum over
    t of the valid j), dX and dW (sum over j of the valid t)."""
    p = K // 2
    t = np.arange(L, dtype=np.int64)
    n = np.clip(np.minimum(K, L + p - t) - np.maximum(0, p - t), 0, None).sum()
    return 2 * B * H * int(n)


def bench_config(cfg_name, args, world):
    """The `config` dict -- identical in both arms (the driver compares them)."""
    B, H, L, K = CONFIGS[cfg_name]
    strong = bool(args.global_batch)
    gb = args.global_batch if strong else B * world
    return {"workload": WORKLOAD[cfg_name], "name": cfg_name, "B": gb, "H": H, "L": L, "K": K,
            "global_batch": gb, "B_per_gpu": (-(-gb // world) if strong else B), "n_gpus": world,
            "scaling": "strong" if strong else "weak", "mode": args.mode, "dw_scheme": args.scheme,
            "bytes_per_step": step_bytes(gb, H, L, K),
            "value_def": "compulsory HBM bytes of the step (20*B*H*L + 12*H*K) / step time"}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(config_name):
    """Per-launch DRAM bytes of the dominant kernels from the committed ncu
    --set full summary (profiles/ncu_summary.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            return json.load(f).get(config_name)
    except Exception:
        return None


def pcie_probe(dev, nbytes=1 << 30, reps=3):
    """Pinned host <-> device copy rates (GB/s): H2D alone, D2H alone, and both
    directions at once on two streams -- the roof of the e2e number."""
    import torch

    n = nbytes // 4
    hs = torch.empty(n, dtype=torch.float32, pin_memory=True)
    hd = torch.empty(n, dtype=torch.float32, pin_memory=True)
    da = torch.empty(n, dtype=torch.float32, device=dev)
    db = torch.empty(n, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(fn):
        best = float("inf")
        for _ in range(reps):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize(dev)
            best = min(best, time.perf_counter() - t0)
        return best

    def h2d():
        with torch.cuda.stream(s1):
            da.copy_(hs, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            hd.copy_(db, non_blocking=True)

    def both():
        h2d()
        d2h()

    t_h, t_d, t_b = timed(h2d), timed(d2h), timed(both)
    del hs, hd, da, db
    return {"h2d_gbs": round(nbytes / t_h / 1e9, 1), "d2h_gbs": round(nbytes / t_d / 1e9, 1),
            "bidir_gbs": round(2 * nbytes / t_b / 1e9, 1)}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[2:6]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU legs (oracle/_ref = the reference's own conv_core.cpp)

def _ref_impl():
    from oracle.oracle import Oracle, Reference, reference_available
    impl = Reference() if reference_available() else Oracle()
    return impl, ("reference" if isinstance(impl, Reference) else "port")


def _ref_step(impl, x, k, gy, K, mode, threads):
    """One step of the reference CPU implementation (default dW scheme
    Sequential, src/conv_core.cpp:98-111) on a channel slice."""
    from oracle.oracle import SEQUENTIAL
    t0 = time.perf_counter()
    impl.forward(x, k, mode, threads=threads)
    impl.backward_input(gy, k, mode, threads=threads)
    impl.backward_weight(gy, x, K, SEQUENTIAL, 0, mode, threads=threads)
    return time.perf_counter() - t0


def cpu_sample(cfg, threads, mode, budget_s=12.0):
    """Time fwd + dX + dW of the reference CPU implementation on a channel
    sample of the workload (all B rows), fanned out over `threads` host
    threads.  Returns (GB/s of the step's compulsory bytes, full-step seconds
    extrapolated to all H channels, sample text, kind)."""
    from oracle.oracle import Oracle
    B, H, L, K = cfg
    impl, kind = _ref_impl()
    o = Oracle()

    def run(hs):
        x, k, gy = o.fill_inputs(7, B, hs, L, K)
        return _ref_step(impl, x, k, gy, K, mode, threads)

    hs = min(H, max(1, threads))
    t = run(hs)
    while t < budget_s / 4 and hs < H:  # grow the sample to a measurable size
        hs = min(H, hs * 2)
        t = run(hs)
    if t < budget_s / 2 and hs < H:
        hs = min(H, max(hs, int(hs * (budget_s / 2) / max(t, 1e-3))))
        t = run(hs)
    mname = "Separate" if mode == 0 else "Fused"
    sample = (f"{hs} of {H} channels (all B={B} rows, L={L}, K={K}), fwd+dX+dW(sequential), "
              f"MulAddMode::{mname}, {threads} threads channel-sliced, {kind} build; full-step time "
              f"extrapolated x{H / hs:.1f}")
    return step_bytes(B, hs, L, K) / t / 1e9, t * H / hs, sample, kind


def run_reference(args, cfg_name, cfg):
    """The reference arm: the reference's own conv_core.cpp on the host cores,
    the same config dict, metric and bytes as this repo's arm."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    B, H, L, K = cfg
    mode = 1 if args.mode == "fused" else 0
    impl, kind = _ref_impl()
    from oracle.oracle import Oracle
    # size the per-step channel sample so warmup + steps fit in ~2 minutes
    _, full_s, _, _ = cpu_sample(cfg, threads, mode, budget_s=4.0)
    per_channel = full_s / H
    total_steps = args.steps + args.warmup
    hs = int(max(1, min(H, 100.0 / total_steps / max(per_channel, 1e-6))))
    x, k, gy = Oracle().fill_inputs(7, B, hs, L, K)
    times = []
    for i in range(total_steps):
        t = _ref_step(impl, x, k, gy, K, mode, threads)
        if i >= args.warmup:
            times.append(t)
    t = sum(times) / len(times)
    gbs = step_bytes(B, hs, L, K) / t / 1e9
    # side number: the other MulAddMode (Fused is a libm fma call in the
    # reference's Release build, ~2.5-3x slower than Separate)
    other = 1 - mode
    t_other = _ref_step(impl, x, k, gy, K, other, threads)
    mname = "Separate" if mode == 0 else "Fused"
    sample = (f"{hs} of {H} channels per step (all B={B} rows), fwd+dX+dW(sequential), MulAddMode::{mname}, "
              f"{threads} threads channel-sliced, {kind} build")
    conf = bench_config(cfg_name, args, world)
    gb = conf["global_batch"]
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * H / hs * gb / B * 1e3, 3), "higher_is_better": True,
        "scaling": conf["scaling"], "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": conf,
        "ms_per_step_note": f"extrapolated from {hs} of {H} channels and {B} rows to the whole global batch",
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "side": {"mode": "fused" if other else "separate",
                 "value": round(step_bytes(B, hs, L, K) / t_other / 1e9, 4), "unit": "GB/s",
                 "note": "one step of the same sample in the other MulAddMode"},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm

def run_ours(args, cfg_name, cfg):
    import torch
    import torch.distributed as dist

    import paper_2604_25422_b200 as ks

    for kv in args.opt:
        name, val = kv.split("=")
        ks.set_option(name, int(val))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world == 1 and args.gpus > 1:
        print("bench.py: --gpus N>1 must be launched under torchrun", file=sys.stderr)
        return 2
    # --transport host: the ranks' plumbing is a gloo group and the dW combine
    # runs over the library's host communicator, so ranks may share a GPU
    # (this is how the N > 1 path of this script is exercised on one B200;
    # NCCL refuses two ranks on one device)
    host_tx = args.transport == "host"
    local_dev = local % max(1, torch.cuda.device_count()) if host_tx else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if host_tx:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    red_dev = torch.device("cpu") if host_tx else dev  # where the timing max-reductions live
    Bc, H, L, K = cfg
    conf = bench_config(cfg_name, args, world)
    B_total = conf["global_batch"]
    if args.global_batch:  # strong scaling: this rank's contiguous rows of the global batch
        b0, B = ks.shard_rows(B_total, world, rank)
    else:  # weak scaling: every rank the config's batch
        b0, B = rank * Bc, Bc
    mode = ks.FUSED if args.mode == "fused" else ks.SEPARATE
    scheme = {"hierarchical": ks.HIERARCHICAL, "pairwise": ks.PAIRWISE}[args.scheme]

    comm = peer = None
    if world > 1 and host_tx:
        def _allgather(data: bytes):
            t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return [o.numpy().tobytes() for o in out]
        comm = ks.Comm.host(world, rank, _allgather)
    elif world > 1:
        uid = [ks.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = ks.Comm(uid[0], world, rank)
    if comm is not None:
        if args.combine == "peer" and scheme == ks.HIERARCHICAL:
            # NVLink peer-memory combine fused into dW (global plan: = the 1-GPU bits when shards align)
            peer = comm.peer(B, H, L, K, B_total=B_total)

    x, k, gy = ks.make_inputs(args.seed, B, H, L, K, device=dev, b0=b0, B_total=B_total)
    y = torch.empty_like(x)
    dx = torch.empty_like(gy)
    dk = torch.empty((H, K), dtype=torch.float32, device=dev)
    ws = torch.empty(max(1, ks.workspace_bytes(B, H, L, K, scheme) // 4), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def run_fwd():
        ks.forward(x, k, mode, out=y)

    def run_dx():
        ks.backward_input(gy, k, mode, out=dx)

    def run_dw():
        if peer is not None:  # stage 1 + fused signal/wait/combine over peer memory
            peer.backward_weight(gy, x, K, mode, out=dk, B_total=B_total)
        else:
            ks.backward_weight(gy, x, K, scheme, 0, mode, out=dk, workspace=ws)

    def run_bwd():
        ks.backward(gy, x, k, mode, out=(dx, dk), workspace=ws)

    fused_bwd = args.bwd == "fused" and peer is None and scheme == ks.HIERARCHICAL
    # split step (gives the per-path table) and the step proper (forward, then
    # the layer's backward in ONE call where it fuses): each path's launches
    # are captured once into a CUDA graph and replayed, so the timed region
    # holds device work only.  The NCCL / peer dW combine stays eager.
    split_fns = [run_fwd, run_dx, run_dw]
    step_fns = [run_fwd, run_bwd] if fused_bwd else list(split_fns)
    launches = {}  # launches of our kernels per call of each path

    def count(fn):
        c0 = ks.launch_count()
        fn()
        return ks.launch_count() - c0

    clk = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        for fn in split_fns + step_fns[1:]:
            fn()
    torch.cuda.synchronize()
    use_graphs = not args.no_graphs and peer is None
    graphs = {}
    if use_graphs:
        try:
            for fn in set(split_fns + step_fns):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    launches[fn] = count(fn)
                graphs[fn] = g
        except Exception as exc:  # capture unsupported here: stay eager, say so
            print(f"bench.py: CUDA graph capture failed ({exc}); timing eager launches", file=sys.stderr)
            graphs = {}
            torch.cuda.synchronize()
    if not graphs:
        for fn in set(split_fns + step_fns):
            launches[fn] = count(fn)
    # the whole step (forward, then the backward) as ONE graph as well: a
    # training loop replays its step once, so the step time below carries one
    # graph launch, not one per path (config 1: ~8 us per replay)
    step_graph = None
    if graphs:
        try:
            step_graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(step_graph):
                for fn in step_fns:
                    fn()
        except Exception as exc:
            print(f"bench.py: whole-step graph capture failed ({exc}); the step time uses per-path graphs",
                  file=sys.stderr)
            step_graph = None
    torch.cuda.synchronize()
    play = {fn: (graphs[fn].replay if fn in graphs else fn) for fn in set(split_fns + step_fns)}

    def run_step():
        step_graph.replay()

    if step_graph is not None:
        play[run_step] = run_step

    def combine():
        if comm is not None and peer is None:
            comm.allreduce_dw(dk)

    # working sets that fit in L2 (126 MB; configs 1 and 2) get L2 flushed
    # before every timed step by writing a 512 MB buffer, outside the timed
    # events; larger ones stream from HBM anyway
    flush = None
    if 4 * B * H * L * 2 < 4 * 126e6:
        flush = torch.empty(128 << 20, dtype=torch.float32, device=dev)

    def timed(fns, with_combine):
        """Times args.steps steps of fns (+ combine): per-step event splits and
        the whole-loop time (flushes excluded)."""
        for _ in range(args.warmup):
            for fn in fns:
                play[fn]()
            combine()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        n = len(fns) + 2
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n)] for _ in range(args.steps)]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(float(i))
            for j, fn in enumerate(fns):
                evs[i][j].record(stream)
                play[fn]()
            evs[i][len(fns)].record(stream)
            if with_combine:
                combine()
            evs[i][len(fns) + 1].record(stream)
        end.record(stream)
        torch.cuda.synchronize()
        per = np.array([[e[j].elapsed_time(e[j + 1]) for j in range(n - 1)] for e in evs])
        total = start.elapsed_time(end) if flush is None else float(sum(e[0].elapsed_time(e[-1]) for e in evs))
        return per, total

    per_split, ms_split_total = timed(split_fns, True)
    per_step, ms_total = (per_split, ms_split_total) if not fused_bwd else timed(step_fns, True)
    if step_graph is not None:  # the step time proper: one replay of the whole step per step
        _, ms_total = timed([run_step], True)
    clk.__exit__(None, None, None)
    split_mean = per_split.mean(axis=0)  # fwd, dX, dW, combine
    step_mean = per_step.mean(axis=0)    # fwd, bwd (or dX, dW), combine
    if world > 1:
        t = torch.tensor([ms_total] + split_mean.tolist() + step_mean.tolist(), dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        v = t.cpu().numpy()
        ms_total, split_mean, step_mean = float(v[0]), v[1:1 + len(split_mean)], v[1 + len(split_mean):]
    ms_step = ms_total / args.steps

    if args.timing_log and rank == 0:
        # the reference's timing-log schema (src/timing_log.cpp:44-97): one row
        # per path per timed step; conv_total = fwd + bwd_in + bwd_k
        with open(args.timing_log, "w") as f:
            f.write(f"# kernelscope timing log from the B200 library (bench.py), {cfg_name}; "
                    f"variant {args.timing_variant}\n")
            f.write("variant,path,runtime_ms,run_id\n")
            for i, row in enumerate(per_split):
                for name, v in zip(("fwd", "bwd_in", "bwd_k"), row[:3]):
                    f.write(f"{args.timing_variant},{name},{v:.6f},{i}\n")
                f.write(f"{args.timing_variant},conv_total,{float(sum(row[:3])):.6f},{i}\n")

    pb = path_bytes(B, H, L, K)
    value = step_bytes(B_total, H, L, K) / (ms_step * 1e-3) / 1e9
    peak, peak_kind = measured_peaks()
    names = ["fwd", "dX", "dW"]
    paths = {}
    for i, n in enumerate(names):
        gbs = pb / (split_mean[i] * 1e-3) / 1e9
        fl = path_flops(B, H, L, K) / (split_mean[i] * 1e-3) / 1e12
        ufl = useful_flops(B, H, L, K) / (split_mean[i] * 1e-3) / 1e12
        paths[n] = {"ms": round(float(split_mean[i]), 4), "GB_s": round(gbs, 1),
                    "frac_hbm_measured": round(gbs / peak, 4), "frac_hbm_8TBs": round(gbs / 8000, 4),
                    "TFLOP_s_paper": round(fl, 2), "TFLOP_s_useful": round(ufl, 2)}
    if world > 1:
        comb_ms = float(step_mean[-1]) if peer is None else None
        paths["dW_combine"] = {"ms": None if comb_ms is None else round(comb_ms, 4), "bytes": 4 * H * K,
                               "kind": "peer-memory (fused into dW)" if peer is not None else "ncclAllReduce",
                               "share_of_step": None if comb_ms is None else round(comb_ms / ms_step, 4)}
    fused_kernel = fused_bwd and L % 32 == 0 and L >= 2048 and K <= 16
    if fused_bwd:
        # logical bytes of the two paths it replaces vs the bytes it moves
        # (fused kernel: read gy + x, write dx = 12 B per element; else 16)
        moved = (12 if fused_kernel else 16) * B * H * L + 8 * H * K
        paths["bwd_fused"] = {"ms": round(float(step_mean[1]), 4),
                              "GB_s_logical": round(2 * pb / (step_mean[1] * 1e-3) / 1e9, 1),
                              "bytes_moved": moved,
                              "GB_s_moved": round(moved / (step_mean[1] * 1e-3) / 1e9, 1),
                              "frac_hbm_measured": round(moved / (step_mean[1] * 1e-3) / 1e9 / peak, 4),
                              "fused_kernel": fused_kernel}
    dom = int(np.argmax(split_mean[:3]))
    traffic = ncu_traffic(cfg_name)
    dom_traffic = None
    if traffic and names[dom] in traffic:
        dom_traffic = traffic[names[dom]].get("dram_bytes")
    achieved = pb / (split_mean[dom] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": dom_traffic,
                "kernel": names[dom], "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": pb,
                "note": "achieved = (8*B*H*L + 4*H*K) bytes / mean CUDA-event duration of the path"}
    if fused_kernel and step_mean[1] > step_mean[0]:
        # the step's dominant kernel is the fused backward: its algorithmic
        # (compulsory) bytes are read gy + x, write dx, read k, write dk
        fb = paths["bwd_fused"]["bytes_moved"]
        ach = fb / (step_mean[1] * 1e-3) / 1e9
        bt = traffic.get("bwd", {}).get("dram_bytes") if traffic else None
        roofline = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 4), "traffic": bt, "kernel": "bwd_fused (dX + dW, one pass)",
                    "peak_kind": peak_kind, "algorithmic_bytes_per_launch": fb,
                    "note": "achieved = (12*B*H*L + 8*H*K) compulsory bytes / mean CUDA-event duration; "
                            "per-path split numbers in `paths`"}
    # long K is FP32-FMA-bound (paper arithmetic intensity K/4 FLOP/B above the
    # ridge): report against the FP32 roof measured in-process instead
    fp32 = None
    if K / 4.0 > 12.0:
        import ctypes
        c = ctypes.c_double(0.0)
        if ks.lib().ks_probe_fp32_tflops(ctypes.byref(c)) == 0:
            fp32 = c.value
    if fp32:
        # the FP32 roof in useful FLOPs per path: FMA pipe at 2 FLOP per
        # instruction.  Forward / dX in Separate mode need two instructions per
        # tap (FMUL + FADD, the reference's two roundings), so their roof is
        # half; HIERARCHICAL dW accumulates with FMA in either mode.
        sep = mode == ks.SEPARATE
        roof = {"fwd": fp32 / 2 if sep else fp32, "dX": fp32 / 2 if sep else fp32, "dW": fp32}
        fl = path_flops(B, H, L, K)
        ufl = useful_flops(B, H, L, K)
        ach = ufl / (split_mean[dom] * 1e-3) / 1e12
        roofline = {"bound": "fp32", "achieved": round(ach, 2), "peak": round(roof[names[dom]], 2),
                    "unit": "TFLOP/s", "frac": round(ach / roof[names[dom]], 4), "traffic": dom_traffic,
                    "kernel": names[dom],
                    "peak_kind": "measured in-process (ks_probe_fp32_tflops: FFMA loop on all SMs)"
                                 + (", halved for a Separate-mode stencil (FMUL + FADD per tap)"
                                    if sep and names[dom] != "dW" else ""),
                    "fp32_fma_peak": round(fp32, 2),
                    "algorithmic_flops_per_launch": ufl, "paper_flops_per_launch": fl,
                    "frac_paper_flops": round(fl / (split_mean[dom] * 1e-3) / 1e12 / roof[names[dom]], 4),
                    "note": "compute-bound (K/4 FLOP/B > ridge); achieved = useful FLOPs (2 x taps that touch "
                            "the row, SURVEY 8(d)) / mean CUDA-event duration of the path; the paper's "
                            "2*B*H*L*K also counts taps on the zero padding (frac_paper_flops); HBM GB/s "
                            "per path in `paths`"}
        for n in names:
            paths[n]["frac_fp32_roof"] = round(paths[n]["TFLOP_s_useful"] / roof[n], 4)
            paths[n]["frac_fp32_paper_flops"] = round(paths[n]["TFLOP_s_paper"] / roof[n], 4)
    # our kernels launched inside the two timed loops (counted by the library
    # at capture / launch time: ks_launch_count)
    gpu_launches = args.steps * (sum(launches[f] for f in split_fns) +
                                 (sum(launches[f] for f in step_fns) if fused_bwd else 0) +
                                 (sum(launches[f] for f in step_fns) if step_graph is not None else 0))

    # ---- end to end from pinned host memory (H2D / D2H inside the timed region) ----
    e2e = e2e_step = None
    e2e_note = None
    if not args.no_e2e:
        # every rank pins x, gy, y, dx on the same host: skip (and say so) when
        # the node's free RAM cannot hold them, instead of failing the run
        need = world * 4 * 4 * B * H * L
        try:
            import psutil
            avail = psutil.virtual_memory().available
        except Exception:
            avail = None
        if avail is not None and need > 0.8 * avail:
            e2e_note = f"skipped: {world} ranks x 4 pinned tensors = {need / 1e9:.0f} GB > 80% of free host RAM"
    if not args.no_e2e and e2e_note is None:
        xh = torch.empty((B, H, L), dtype=torch.float32, pin_memory=True)
        gyh = torch.empty_like(xh, pin_memory=True)
        yh = torch.empty_like(xh, pin_memory=True)
        dxh = torch.empty_like(xh, pin_memory=True)
        kh = torch.empty((H, K), dtype=torch.float32, pin_memory=True)
        dkh = torch.empty((H, K), dtype=torch.float32, pin_memory=True)
        xh.copy_(x)
        gyh.copy_(gy)
        kh.copy_(k)
        xn, gyn, yn, dxn, kn, dkn = (t.numpy() for t in (xh, gyh, yh, dxh, kh, dkh))
        del y, dx
        torch.cuda.empty_cache()
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        tb, kb = 4 * B * H * L, 4 * H * K
        pcie = pcie_probe(dev)

        def host_calls():  # the reference's three value-type calls, each through its own host entry
            ks.forward(xn, kn, mode, out=yn)
            ks.backward_input(gyn, kn, mode, out=dxn)
            ks.backward_weight(gyn, xn, K, scheme, 0, mode, out=dkn)

        def host_step():  # the library's one-call step: x and gy cross PCIe once
            ks.step_host(xn, kn, gyn, scheme=scheme, mode=mode, out=(yn, dxn, dkn))

        def measure(fn, h2d, d2h, path):
            fn()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                fn()
            t_host = (time.perf_counter() - t0) / e2e_steps
            if world > 1:
                tt = torch.tensor([t_host], dtype=torch.float64, device=red_dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t_host = float(tt[0])
            # the e2e roof: the step's PCIe bytes at the link's measured rates
            # (H2D and D2H overlap on separate copy engines)
            bound_s = max(h2d / (pcie["h2d_gbs"] * 1e9), d2h / (pcie["d2h_gbs"] * 1e9),
                          (h2d + d2h) / (pcie["bidir_gbs"] * 1e9))
            return {"value": round(step_bytes(B_total, H, L, K) / t_host / 1e9, 2), "unit": "GB/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": round(t_host * 1e3, 2), "steps": e2e_steps, "path": path,
                    "pcie": dict(pcie, bound_ms=round(bound_s * 1e3, 2), frac=round(bound_s / t_host, 4))}

        e2e = measure(host_calls, 4 * tb + 2 * kb, 2 * tb + kb,
                      "drop-in: ks_dwconv1d_{fwd,dx,dw}_f32_host (the reference's three value-type calls: "
                      "x, gy, gy, x up; y, dx, dk down), pinned host buffers, wall clock")
        e2e_step = measure(host_step, 2 * tb + kb, 2 * tb + kb,
                           "ks_dwconv1d_step_f32_host (one call: x, gy up once; y, dx, dk down), pinned host "
                           "buffers, wall clock")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        gbs, _, sample, kind = cpu_sample(cfg, threads, 1 if args.mode == "fused" else 0)
        cpu = {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": kind, "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": conf["scaling"], "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference splitmix64 stream, generated on device)",
            "config": conf,
            "run": {"parallelism": f"batch-shard dp{world}" + (
                        "" if world == 1 else " + dW combine fused over peer memory" if peer is not None
                        else " + NCCL dW allreduce" if not host_tx else " + dW allreduce over the host communicator"),
                    "transport": args.transport,
                    "gpus_visible": torch.cuda.device_count(),
                    "rows_this_rank": B,
                    "l2": "inputs larger than L2 (no flush)" if flush is None
                          else "L2 flushed before every timed step (512 MB write, untimed)",
                    "cuda_graphs": bool(graphs),
                    **({"options": list(args.opt)} if args.opt else {}),
                    "step_timing": "one CUDA-graph replay per step (fwd + bwd)" if step_graph is not None
                                   else "per-path launches",
                    "step_bwd": "fused (ks_dwconv1d_bwd_f32)" if fused_bwd else "split (dx, dw calls)",
                    "frac_hbm_measured": round(value / world / peak, 4), "frac_hbm_8TBs": round(value / world / 8000, 4)},
            "paths": paths,
            "step_paths_ms": {n: round(float(v), 4) for n, v in zip(
                (["fwd", "bwd"] if fused_bwd else ["fwd", "dX", "dW"]) + ["combine"], step_mean)},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            **({"e2e_step": e2e_step} if e2e_step else {}),
            **({"e2e_note": e2e_note} if e2e_note else {}),
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if peer is not None:
        if peer.timed_out():
            print("bench.py: a peer dW combine timed out (dk is NaN)", file=sys.stderr)
            return 3
        peer.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="config3")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="strong scaling: fixed global batch sharded over the ranks (ks_shard_rows); "
                         "default: weak scaling with the config's batch on every rank")
    ap.add_argument("--mode", choices=["separate", "fused"], default="separate",
                    help="MulAddMode (the reference's default is Separate)")
    ap.add_argument("--scheme", choices=["hierarchical", "pairwise"], default="hierarchical")
    ap.add_argument("--combine", choices=["nccl", "peer"], default="nccl",
                    help="N>1 dW combine: one allreduce, or the fused NVLink peer-memory kernel")
    ap.add_argument("--transport", choices=["nccl", "host"], default="nccl",
                    help="N>1 plumbing: NCCL (one GPU per rank), or gloo + the library's host communicator "
                         "(ranks may share a GPU: the N>1 code path on a 1-GPU box)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--timing-log", default=None,
                    help="also write per-step path times in the reference's timing CSV schema")
    ap.add_argument("--timing-variant", default="warp",
                    help="variant column of --timing-log (the reference's parser accepts naive/gmc/shared/warp)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graphs", action="store_true", help="launch each path eagerly instead of replaying CUDA graphs")
    ap.add_argument("--opt", action="append", default=[],
                    help="library tuning option name=value (ks_set_option; A/B runs, recorded in the line)")
    ap.add_argument("--bwd", choices=["fused", "split"], default="fused",
                    help="step backward: one ks_dwconv1d_bwd_f32 call (dX + dW in one pass) or the two calls")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, args.config, cfg)
    return run_ours(args, args.config, cfg)


if __name__ == "__main__":
    sys.exit(main())
