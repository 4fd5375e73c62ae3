#!/usr/bin/env python3
"""Performance-cliff sweep over shapes outside the BASELINE configs: every
path graph-timed at a grid of (L, K) (B, H sized to ~2^27 elements), with
the time the binding roof allows beside it -- max(bytes / HBM, useful FLOPs /
FP32) with the HBM rate of the path's read:write mix (profiles/r02_hbm_mix.txt)
and the FP32 FFMA rate (halved for a Separate-mode stencil: two instructions
per tap).  A low `roof%` flags a shape whose tier is a poor fit.  Not a bench
line.

usage: python tools/roof_sweep.py [--mode separate|fused] [--paths fwd,dx,dw] [--elems 134217728]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_25422_b200 as ks  # noqa: E402

HBM_1TO1, HBM_READ = 6.5e12, 7.3e12   # B/s: fwd / dX stream (1:1), dW (read-only)
FP32 = 72e12                           # FLOP/s, FFMA on all SMs

LS = [48, 128, 256, 500, 1000, 1024, 2048, 4095, 4096, 16384]
KS = [3, 7, 12, 16, 24, 32, 48, 64, 128, 256, 1024, 4096]


def useful_taps(L, K):
    p = K // 2
    tot = 0
    for t in range(L):
        lo, hi = max(0, p - t), min(K, L + p - t)
        tot += max(0, hi - lo)
    return tot  # per row


def timed(fn, reps=5, inner=5):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(inner):
            fn()
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / inner)
    ts = sorted(ts[1:])
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", choices=["separate", "fused"], default="separate")
    ap.add_argument("--paths", default="fwd,dx,dw")
    ap.add_argument("--elems", type=int, default=1 << 27)
    a = ap.parse_args()
    mode = ks.FUSED if a.mode == "fused" else ks.SEPARATE
    paths = a.paths.split(",")
    print(f"mode {a.mode}; per path: ms, roof ms, roof% (binding roof: hbm / fp32)")
    print("shape".ljust(24), *[f"{p:>26}" for p in paths], "  kernel(fwd)")
    for L in LS:
        for K in KS:
            if K > L:
                continue
            H = 64
            B = max(1, a.elems // (H * L))
            x, k, gy = ks.make_inputs(1, B, H, L, K)
            y, dx = torch.empty_like(x), torch.empty_like(x)
            n = B * H * L
            taps = useful_taps(L, K) * B * H
            fns = {"fwd": lambda: ks.forward(x, k, mode, out=y),
                   "dx": lambda: ks.backward_input(gy, k, mode, out=dx),
                   "dw": lambda: ks.backward_weight(gy, x, K, ks.HIERARCHICAL, 0, mode)}
            cells = []
            for p in paths:
                ms = timed(fns[p])
                hbm = 8 * n / (HBM_READ if p == "dw" else HBM_1TO1)
                rate = FP32 / (2 if (p != "dw" and mode == ks.SEPARATE) else 1)
                fp = 2 * taps / rate
                roof = max(hbm, fp) * 1e3
                cells.append(f"{ms:8.3f} {roof:8.3f} {100 * roof / ms:5.0f}% {'h' if hbm >= fp else 'f'}")
            kern = ks.plan("fwd", B, H, L, K, mode=mode)
            kname = kern[-1]["kernel"].split("::")[-1].split("(")[0] if kern else "?"
            print(f"({B},{H},{L},{K})".ljust(24), *[c.rjust(26) for c in cells], " ", kname)
            del x, k, gy, y, dx
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
