#!/usr/bin/env python3
"""bench.py -- S4ConvD depthwise conv1d fwd + dX + dW step on B200.

Metric (BASELINE.json): effective HBM GB/s and % of the HBM roofline per path
(fwd / dX / dW), and fwd+bwd conv time per step.

* A "step" is one pass of the hot path over one batch: y = forward(x,k),
  dx = backward_input(gy,k), dk = backward_weight(gy,x) (+ the dW combine over
  ranks when N > 1), all through the library's C ABI on resident device
  buffers.  Inputs come from the reference's splitmix64 stream generated in
  place on the device.
* Default workload: BASELINE config 3 (B=256, H=512, L=8192, K=7, fp32), the
  largest single-GPU config and the one the north star's roofline targets are
  stated on.  4 GiB per tensor >> 126 MB L2, so no L2 flush is needed.
* value = algorithmic bytes of the three paths (8*B*H*L + 4*H*K each,
  reference src/exec_model.cpp:168-179) over all ranks / device step time
  (CUDA events, max over ranks).  Weak scaling: every rank runs the per-GPU
  batch B, the global batch is B*N, sharded by contiguous batch rows.
* e2e: the same metric through the host-buffer C-ABI entry points
  (ks_dwconv1d_*_host, the reference's value-type API shape) from pinned host
  memory, H2D/D2H inside the timed region.
* --impl reference: the reference's own CPU conv_core.cpp (oracle/_ref, built
  from /root/reference) on the host cores, channel-sliced over threads, on a
  bounded channel sample of the same workload.
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


def path_flops(B, H, L, K):
    return 2 * B * H * L * K  # reference src/analyzer.cpp:36-49


def useful_flops(B, H, L, K):
    """2 x the taps that touch the row: the paper's count includes
    taps on the zero padding, 25% of them at K = L.  Same total for fwd (sum over
    t of the valid j), dX and dW (sum over j of the valid t)."""
    import numpy as np
    p = K // 2
    t = np.arange(L, dtype=np.int64)
    n = np.clip(np.minimum(K, L + p - t) - np.maximum(0, p - t), 0, None).sum()
    return 2 * B * H * int(n)


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

def cpu_sample(cfg, threads, budget_s=12.0, mode=1, reps=1):
    """Time fwd + dX + dW (reference default dW scheme: sequential) of the
    reference CPU implementation on a channel sample of the workload, fanned
    out over `threads` host threads.  Returns (GB/s, seconds, sample dict)."""
    from oracle.oracle import SEQUENTIAL, Reference, reference_available, Oracle
    B, H, L, K = cfg
    impl = Reference() if reference_available() else Oracle()
    kind = "reference" if isinstance(impl, Reference) else "port"

    def run(hs):
        o = Oracle()
        x, k, gy = o.fill_inputs(7, B, hs, L, K)
        t0 = time.perf_counter()
        impl.forward(x, k, mode, threads=threads)
        impl.backward_input(gy, k, mode, threads=threads)
        impl.backward_weight(gy, x, K, SEQUENTIAL, 0, mode, threads=threads)
        return time.perf_counter() - t0

    hs = min(H, max(1, threads))
    t = run(hs)
    while t < budget_s / 4 and hs < H:  # grow the sample to a measurable size
        hs = min(H, hs * 2)
        t = run(hs)
    if t < budget_s / 2 and hs < H:
        hs = min(H, max(hs, int(hs * (budget_s / 2) / max(t, 1e-3))))
        t = run(hs)
    times = [t] + [run(hs) for _ in range(reps - 1)]
    t = min(times)
    bytes_ = 3 * path_bytes(B, hs, L, K)
    sample = (f"{hs} of {H} channels (all B={B} rows, L={L}, K={K}), fwd+dX+dW(sequential), "
              f"{threads} threads channel-sliced, {kind} build; full-step time extrapolated x{H / hs:.1f}")
    return bytes_ / t / 1e9, t * H / hs, sample, kind


def run_reference(args, cfg_name, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    B, H, L, K = cfg
    from oracle.oracle import SEQUENTIAL, Reference, reference_available, Oracle
    impl = Reference() if reference_available() else Oracle()
    kind = "reference" if isinstance(impl, Reference) else "port"
    # size the per-step channel sample so warmup+steps fit in ~2 minutes
    _, full_s, _, _ = cpu_sample(cfg, threads, budget_s=4.0)
    per_channel = full_s / H
    total_steps = args.steps + args.warmup
    hs = int(max(1, min(H, 110.0 / total_steps / max(per_channel, 1e-6))))
    o = Oracle()
    x, k, gy = o.fill_inputs(7, B, hs, L, K)
    times = []
    for i in range(total_steps):
        t0 = time.perf_counter()
        impl.forward(x, k, 1, threads=threads)
        impl.backward_input(gy, k, 1, threads=threads)
        impl.backward_weight(gy, x, K, SEQUENTIAL, 0, 1, threads=threads)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    gbs = 3 * path_bytes(B, hs, L, K) / t / 1e9
    sample = (f"{hs} of {H} channels per step (all B={B} rows), fwd+dX+dW(sequential, Fused), "
              f"{threads} threads channel-sliced")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * H / hs * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD[cfg_name], "name": cfg_name, "B": B, "H": H, "L": L,
                   "K": K, "global_batch": B, "ms_per_step_note": "extrapolated to all H channels"},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm

def run_ours(args, cfg_name, cfg):
    import torch
    import torch.distributed as dist

    import paper_2604_25422_b200 as ks

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            print("bench.py: --gpus N>1 must be launched under torchrun", file=sys.stderr)
            return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    B, H, L, K = cfg
    mode = ks.FUSED if args.mode == "fused" else ks.SEPARATE
    scheme = {"hierarchical": ks.HIERARCHICAL, "pairwise": ks.PAIRWISE}[args.scheme]

    comm = peer = None
    if world > 1:
        uid = [ks.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = ks.Comm(uid[0], world, rank)
        if args.combine == "peer" and scheme == ks.HIERARCHICAL:
            peer = comm.peer(B, H, L, K)  # NVLink peer-memory combine fused into dW

    # inputs: rows [rank*B, rank*B+B) of the (B*world)-row problem, generated in place
    x, k, gy = ks.make_inputs(args.seed, B, H, L, K, device=dev, b0=rank * B, B_total=B * world)
    y = torch.empty_like(x)
    dx = torch.empty_like(gy)
    dk = torch.empty((H, K), dtype=torch.float32, device=dev)
    ws = torch.empty(max(1, ks.workspace_bytes(B, H, L, K, scheme) // 4), dtype=torch.float32,
                     device=dev)
    stream = torch.cuda.current_stream(dev)

    def run_fwd():
        ks.forward(x, k, mode, out=y)

    def run_dx():
        ks.backward_input(gy, k, mode, out=dx)

    def run_dw():
        if peer is not None:  # stage 1 + fused signal/wait/combine over peer memory
            peer.backward_weight(gy, x, K, mode, out=dk)
        else:
            ks.backward_weight(gy, x, K, scheme, 0, mode, out=dk, workspace=ws)

    paths_fn = [run_fwd, run_dx, run_dw]

    def step(ev=None):
        for i, fn in enumerate(paths_fn):
            if ev:
                ev[i].record(stream)
            fn()
        if ev:
            ev[3].record(stream)
        if comm is not None and peer is None:
            comm.allreduce_dw(dk)
        if ev:
            ev[4].record(stream)

    # the clock sampler (an nvidia-smi child) starts before the warm-up so its
    # process start-up cannot stall the host inside the timed region
    clk = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # each path's launches (tap staging, kernel(s), stream-ordered scratch) are
    # captured once into a CUDA graph and replayed: the timed region then holds
    # device work only, not the host's per-call launch overhead (which decides
    # launch-bound configs such as config 1).  The NCCL dW combine stays eager.
    graphs = None
    if not args.no_graphs and peer is None:
        try:
            graphs = []
            for fn in paths_fn:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    fn()
                graphs.append(g)
        except Exception as exc:  # capture unsupported here: stay eager, say so
            print(f"bench.py: CUDA graph capture failed ({exc}); timing eager launches", file=sys.stderr)
            graphs = None
            torch.cuda.synchronize()
        if graphs is not None:
            paths_fn = [g.replay for g in graphs]
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    # working sets that fit in L2 (126 MB; configs 1 and 2) get L2 flushed
    # before every timed step by writing a 512 MB buffer, outside the timed
    # events; larger ones stream from HBM anyway
    flush = None
    if 4 * B * H * L * 2 < 4 * 126e6:
        flush = torch.empty(128 << 20, dtype=torch.float32, device=dev)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for i in range(args.steps):
        if flush is not None:
            flush.fill_(float(i))
        step(evs[i])
    end.record(stream)
    torch.cuda.synchronize()

    # The step proper: forward, then the layer's backward in ONE call
    # (ks_dwconv1d_bwd_f32: dX and dW from a single pass over gy and x where
    # the fused kernel applies, bitwise the same dx / dk as the split calls
    # timed above, which give the per-path table).
    fused_bwd = args.bwd == "fused" and peer is None and scheme == ks.HIERARCHICAL
    fevs = None
    if fused_bwd:
        def run_bwd():
            ks.backward(gy, x, k, mode, out=(dx, dk), workspace=ws)

        bwd_fn = run_bwd
        if graphs is not None:
            gb = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gb):
                run_bwd()
            graphs.append(gb)
            bwd_fn = gb.replay

        def fstep(ev=None):
            if ev:
                ev[0].record(stream)
            paths_fn[0]()
            if ev:
                ev[1].record(stream)
            bwd_fn()
            if ev:
                ev[2].record(stream)
            if comm is not None:
                comm.allreduce_dw(dk)
            if ev:
                ev[3].record(stream)

        for _ in range(args.warmup):
            fstep()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        fevs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
        fstart = torch.cuda.Event(enable_timing=True)
        fend = torch.cuda.Event(enable_timing=True)
        fstart.record(stream)
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(float(i))
            fstep(fevs[i])
        fend.record(stream)
        torch.cuda.synchronize()
    clk.__exit__(None, None, None)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    per = np.array([[e[i].elapsed_time(e[i + 1]) for i in range(4)] for e in evs])  # steps x 4
    per_mean = per.mean(axis=0)
    # the step is first path start -> combine end, summed over steps (flushes excluded)
    ms_total = start.elapsed_time(end) if flush is None else float(
        sum(e[0].elapsed_time(e[4]) for e in evs))
    fper_mean = np.zeros(3)
    if fused_bwd:
        fper_mean = np.array([[e[i].elapsed_time(e[i + 1]) for i in range(3)] for e in fevs]).mean(axis=0)
        ms_total = fstart.elapsed_time(fend) if flush is None else float(
            sum(e[0].elapsed_time(e[3]) for e in fevs))
    if world > 1:
        t = torch.tensor([ms_total] + per_mean.tolist() + fper_mean.tolist(), dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total, per_mean, fper_mean = float(t[0]), t[1:5].cpu().numpy(), t[5:8].cpu().numpy()
    ms_step = ms_total / args.steps

    if args.timing_log and rank == 0:
        # the reference's timing-log schema (src/timing_log.cpp:44-97): one row
        # per path per timed step; conv_total = fwd + bwd_in + bwd_k
        with open(args.timing_log, "w") as f:
            f.write("# kernelscope timing log from the B200 library (bench.py); variant b200_tma\n")
            f.write("variant,path,runtime_ms,run_id\n")
            for i, row in enumerate(per):
                for name, v in zip(("fwd", "bwd_in", "bwd_k"), row[:3]):
                    f.write(f"b200_tma,{name},{v:.6f},{i}\n")
                f.write(f"b200_tma,conv_total,{float(sum(row[:3])):.6f},{i}\n")

    pb = path_bytes(B, H, L, K)
    value = world * 3 * pb / (ms_step * 1e-3) / 1e9
    peak, peak_kind = measured_peaks()
    names = ["fwd", "dX", "dW"]
    paths = {}
    for i, n in enumerate(names):
        gbs = pb / (per_mean[i] * 1e-3) / 1e9
        fl = path_flops(B, H, L, K) / (per_mean[i] * 1e-3) / 1e12
        ufl = useful_flops(B, H, L, K) / (per_mean[i] * 1e-3) / 1e12
        paths[n] = {"ms": round(float(per_mean[i]), 4), "GB_s": round(gbs, 1),
                    "frac_hbm_measured": round(gbs / peak, 4), "frac_hbm_8TBs": round(gbs / 8000, 4),
                    "TFLOP_s_paper": round(fl, 2), "TFLOP_s_useful": round(ufl, 2)}
    if world > 1:
        paths["dW_allreduce"] = {"ms": round(float(per_mean[3]), 4), "bytes": 4 * H * K}
    if fused_bwd:
        # logical bytes of the two paths it replaces vs the bytes it moves
        # (fused kernel: read gy + x, write dx = 12 B per element; else 16)
        fused_kernel = L % 32 == 0 and L >= 2048 and K <= 16
        moved = (12 if fused_kernel else 16) * B * H * L + 8 * H * K
        paths["bwd_fused"] = {"ms": round(float(fper_mean[1]), 4),
                              "GB_s_logical": round(2 * pb / (fper_mean[1] * 1e-3) / 1e9, 1),
                              "bytes_moved": moved,
                              "GB_s_moved": round(moved / (fper_mean[1] * 1e-3) / 1e9, 1),
                              "frac_hbm_measured": round(moved / (fper_mean[1] * 1e-3) / 1e9 / peak, 4),
                              "fused_kernel": fused_kernel}
    dom = int(np.argmax(per_mean[:3]))
    traffic = ncu_traffic(cfg_name)
    dom_traffic = None
    if traffic and names[dom] in traffic:
        dom_traffic = traffic[names[dom]].get("dram_bytes")
    achieved = pb / (per_mean[dom] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": dom_traffic,
                "kernel": names[dom], "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": pb,
                "note": "achieved = (8*B*H*L + 4*H*K) bytes / mean CUDA-event duration of the path"}
    if fused_bwd and paths["bwd_fused"]["fused_kernel"] and fper_mean[1] > fper_mean[0]:
        # the step's dominant kernel is the fused backward: its algorithmic
        # (compulsory) bytes are read gy + x, write dx, read k, write dk
        fb = paths["bwd_fused"]["bytes_moved"]
        ach = fb / (fper_mean[1] * 1e-3) / 1e9
        bt = traffic.get("bwd", {}).get("dram_bytes") if traffic else None
        roofline = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 4), "traffic": bt, "kernel": "bwd_fused (dX + dW, one pass)",
                    "peak_kind": peak_kind, "algorithmic_bytes_per_launch": fb,
                    "note": "achieved = (12*B*H*L + 8*H*K) compulsory bytes / mean CUDA-event duration; "
                            "per-path split numbers in `paths`"}
    # long K is FP32-FMA-bound (paper arithmetic intensity K/4 FLOP/B above the
    # ridge): report against the FP32 roof measured in-process instead
    fp32 = C_double = None
    if K / 4.0 > 12.0:
        import ctypes
        C_double = ctypes.c_double(0.0)
        if ks.lib().ks_probe_fp32_tflops(ctypes.byref(C_double)) == 0:
            fp32 = C_double.value
    if fp32:
        fl = path_flops(B, H, L, K)
        ufl = useful_flops(B, H, L, K)
        ach = ufl / (per_mean[dom] * 1e-3) / 1e12
        roofline = {"bound": "fp32", "achieved": round(ach, 2), "peak": round(fp32, 2), "unit": "TFLOP/s",
                    "frac": round(ach / fp32, 4), "traffic": dom_traffic, "kernel": names[dom],
                    "peak_kind": "measured in-process (ks_probe_fp32_tflops: FFMA loop on all SMs)",
                    "algorithmic_flops_per_launch": ufl, "paper_flops_per_launch": fl,
                    "frac_paper_flops": round(fl / (per_mean[dom] * 1e-3) / 1e12 / fp32, 4),
                    "note": "compute-bound (K/4 FLOP/B > ridge); achieved = useful FLOPs (2 x taps that touch "
                            "the row, SURVEY 8(d)) / mean CUDA-event duration of the path; the paper's "
                            "2*B*H*L*K also counts taps on the zero padding (frac_paper_flops); HBM GB/s "
                            "per path in `paths`"}
        for n in names:
            paths[n]["frac_fp32_measured"] = round(paths[n]["TFLOP_s_useful"] / fp32, 4)
            paths[n]["frac_fp32_paper_flops"] = round(paths[n]["TFLOP_s_paper"] / fp32, 4)
    # our kernels per step: fwd and dX = prep_taps + stencil_tma each (TMA path,
    # L % 32 == 0) or one conv_tile_f32; dW = stage 1 + the fixed-order
    # cross-block pass (hierarchical and pairwise alike)
    launches_per_step = (2 * 2 if L % 32 == 0 else 2) + 2
    launches = launches_per_step * args.steps
    if fused_bwd:  # the fused-step loop: fwd (2) + bwd (fused kernel + group sum, or the split 4)
        fused_kernel = L % 32 == 0 and L >= 2048 and K <= 16
        launches += ((2 if L % 32 == 0 else 1) + (2 if fused_kernel else launches_per_step - 2)) * args.steps

    # ---- end to end through the host-buffer C ABI (pinned host memory) ----
    e2e = None
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

        def host_step():
            if args.e2e_path == "step":
                ks.step_host(xn, kn, gyn, scheme=scheme, mode=mode, out=(yn, dxn, dkn))
            else:  # the reference's three value-type calls, each through its own host entry
                ks.forward(xn, kn, mode, out=yn)
                ks.backward_input(gyn, kn, mode, out=dxn)
                ks.backward_weight(gyn, xn, K, scheme, 0, mode, out=dkn)

        host_step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            host_step()
        t_host = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            tt = torch.tensor([t_host], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_host = float(tt[0])
        tb = 4 * B * H * L
        if args.e2e_path == "step":
            h2d, d2h = 2 * tb + 4 * H * K, 2 * tb + 4 * H * K
            path = "ks_dwconv1d_step_f32_host (x, gy up once; y, dx, dk down), pinned host buffers, wall clock"
        else:
            h2d, d2h = 4 * tb + 2 * 4 * H * K, 2 * tb + 4 * H * K
            path = "ks_dwconv1d_{fwd,dx,dw}_f32_host, pinned host buffers, wall clock"
        e2e = {"value": round(world * 3 * pb / t_host / 1e9, 2), "unit": "GB/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(t_host * 1e3, 2), "steps": e2e_steps, "path": path}
        # the e2e roof: the step's PCIe bytes at the link's measured rates
        # (H2D and D2H overlap on separate copy engines)
        pcie = pcie_probe(dev)
        bound_s = max(h2d / (pcie["h2d_gbs"] * 1e9), d2h / (pcie["d2h_gbs"] * 1e9),
                      (h2d + d2h) / (pcie["bidir_gbs"] * 1e9))
        pcie["bound_ms"] = round(bound_s * 1e3, 2)
        pcie["frac"] = round(bound_s / t_host, 4)
        e2e["pcie"] = pcie

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        gbs, _, sample, kind = cpu_sample(cfg, threads)
        cpu = {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": kind,
               "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference splitmix64 stream, generated on device)",
            "config": {"workload": WORKLOAD[cfg_name], "name": cfg_name, "B_per_gpu": B, "H": H,
                       "L": L, "K": K, "global_batch": B * world,
                       "parallelism": f"batch-shard dp{world}" + (
                           "" if world == 1 else " + dW combine fused over NVLink peer memory" if peer is not None
                           else " + NCCL dW allreduce"),
                       "mode": args.mode, "dw_scheme": args.scheme,
                       "l2": "inputs larger than L2 (no flush)" if flush is None
                             else "L2 flushed before every timed step (512 MB write, untimed)",
                       "cuda_graphs": graphs is not None,
                       "step_bwd": "fused (ks_dwconv1d_bwd_f32)" if fused_bwd else "split (dx, dw calls)"},
            "paths": paths, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            **({"e2e_note": e2e_note} if e2e_note else {}),
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if peer is not None:
        peer.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="config3")
    ap.add_argument("--mode", choices=["fused", "separate"], default="fused")
    ap.add_argument("--scheme", choices=["hierarchical", "pairwise"], default="hierarchical")
    ap.add_argument("--combine", choices=["nccl", "peer"], default="nccl",
                    help="N>1 dW combine: one ncclAllReduce, or the fused NVLink peer-memory kernel")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-path", choices=["step", "calls"], default="step")
    ap.add_argument("--timing-log", default=None,
                    help="also write per-step path times in the reference's timing CSV schema")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graphs", action="store_true", help="launch each path eagerly instead of replaying CUDA graphs")
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
