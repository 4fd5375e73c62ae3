#!/usr/bin/env python3
"""Run fwd, dX and dW once per rep at one shape (for ncu captures).

usage: python tools/run_shape.py B H L K [--reps N] [--scheme hierarchical|pairwise]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_25422_b200 as ks  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("shape", type=int, nargs=4)
ap.add_argument("--mode", choices=["separate", "fused"], default="separate")
ap.add_argument("--opt", action="append", default=[], help="tuning option name=value (ks_set_option)")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--scheme", default="hierarchical")
ap.add_argument("--bwd", action="store_true", help="also run the fused backward (ks_dwconv1d_bwd_f32)")
a = ap.parse_args()
B, H, L, K = a.shape
MODE = ks.FUSED if a.mode == "fused" else ks.SEPARATE
for kv in a.opt:
    name, val = kv.split("=")
    ks.set_option(name, int(val))
scheme = {"hierarchical": ks.HIERARCHICAL, "pairwise": ks.PAIRWISE}[a.scheme]
x, k, gy = ks.make_inputs(1, B, H, L, K)
for _ in range(a.reps):
    y = ks.forward(x, k, MODE)
    dx = ks.backward_input(gy, k, MODE)
    dk = ks.backward_weight(gy, x, K, scheme, 0, MODE)
    if a.bwd:
        dx2, dk2 = ks.backward(gy, x, k, MODE)
torch.cuda.synchronize()
print("done", float(y.abs().sum()), float(dx.abs().sum()), float(dk.abs().sum()))
