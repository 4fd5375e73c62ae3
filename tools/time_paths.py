#!/usr/bin/env python3
"""Quick per-path timing at one shape (CUDA events, median of --reps), next to
a device copy of the same bytes (torch copy_, the MEASURED_PEAKS method) --
for A/B sweeps of tuning knobs on the GPU box.  Not a bench line.

usage: python tools/time_paths.py B H L K [--reps N] [--paths fwd,dx,dw,bwd]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_25422_b200 as ks  # noqa: E402


def timed(fn, reps):
    ts = []
    for _ in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts = sorted(ts[2:])
    return ts[len(ts) // 2]


ap = argparse.ArgumentParser()
ap.add_argument("shape", type=int, nargs=4)
ap.add_argument("--mode", choices=["separate", "fused"], default="separate")
ap.add_argument("--opt", action="append", default=[], help="tuning option name=value (ks_set_option)")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--paths", default="fwd,dx,dw,bwd")
a = ap.parse_args()
B, H, L, K = a.shape
MODE = ks.FUSED if a.mode == "fused" else ks.SEPARATE
for kv in a.opt:
    name, val = kv.split("=")
    ks.set_option(name, int(val))
x, k, gy = ks.make_inputs(1, B, H, L, K)
y = torch.empty_like(x)
dx = torch.empty_like(x)
dk = torch.empty((H, K), device="cuda")
n = B * H * L
out = {}
paths = a.paths.split(",")
if "fwd" in paths:
    ms = timed(lambda: ks.forward(x, k, MODE, out=y), a.reps)
    out["fwd"] = (ms, 8 * n / ms / 1e6)
if "dx" in paths:
    ms = timed(lambda: ks.backward_input(gy, k, MODE, out=dx), a.reps)
    out["dx"] = (ms, 8 * n / ms / 1e6)
if "dw" in paths:
    ms = timed(lambda: ks.backward_weight(gy, x, K, ks.HIERARCHICAL, 0, MODE), a.reps)
    out["dw"] = (ms, 8 * n / ms / 1e6)
if "bwd" in paths:
    ms = timed(lambda: ks.backward(gy, x, k, MODE, out=(dx, dk)), a.reps)
    out["bwd"] = (ms, 12 * n / ms / 1e6)
ms = timed(lambda: y.copy_(x), a.reps)
out["copy"] = (ms, 8 * n / ms / 1e6)
print(f"shape {B} {H} {L} {K} env " + " ".join(f"{e}={os.environ[e]}" for e in sorted(os.environ) if e.startswith("KS_")))
for p, (ms, gbs) in out.items():
    print(f"  {p:5s} {ms:9.4f} ms  {gbs:8.1f} GB/s")
