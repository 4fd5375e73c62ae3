#!/usr/bin/env python3
"""ABAB sweep of tuning-option sets over many shapes in ONE process (time_paths.py
starts a process per shape): per (shape, path, option set) the median of the
per-round medians.  Used to place tier thresholds (e.g. which K the register-
window stencil takes, option ldg).  Not a bench line.

usage: python tools/sweep_options.py --shapes "256 512 8192 9;256 512 8192 16" \
           --sets "-;ldg=2" [--paths fwd,dx] [--mode separate|fused] [--rounds 3] [--reps 7]
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


def parse_set(s):
    if s == "-":
        return {}
    return {kv.split("=")[0]: int(kv.split("=")[1]) for kv in s.split(",")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", required=True)
    ap.add_argument("--sets", required=True)
    ap.add_argument("--paths", default="fwd,dx")
    ap.add_argument("--mode", choices=["separate", "fused"], default="separate")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--graph", action="store_true", help="time CUDA-graph replays of --inner calls (small shapes)")
    ap.add_argument("--inner", type=int, default=20, help="calls per graph replay with --graph")
    a = ap.parse_args()
    mode = ks.FUSED if a.mode == "fused" else ks.SEPARATE
    shapes = [tuple(int(v) for v in s.split()) for s in a.shapes.split(";")]
    sets = a.sets.split(";")
    paths = a.paths.split(",")
    res = {}
    for shape in shapes:
        B, H, L, K = shape
        x, k, gy = ks.make_inputs(1, B, H, L, K)
        y, dx = torch.empty_like(x), torch.empty_like(x)
        fns = {"fwd": lambda: ks.forward(x, k, mode, out=y),
               "dx": lambda: ks.backward_input(gy, k, mode, out=dx),
               "dw": lambda: ks.backward_weight(gy, x, K, ks.HIERARCHICAL, 0, mode),
               "bwd": lambda: ks.backward(gy, x, k, mode)}
        for _ in range(a.rounds):
            for s in sets:
                with ks.options(**parse_set(s)):
                    for p in paths:
                        if a.graph:  # options are read at capture time
                            fns[p]()
                            torch.cuda.synchronize()
                            g = torch.cuda.CUDAGraph()
                            with torch.cuda.graph(g):
                                for _ in range(a.inner):
                                    fns[p]()
                            ms = timed(g.replay, a.reps) / a.inner
                        else:
                            ms = timed(fns[p], a.reps)
                        res.setdefault((shape, p, s), []).append(ms)
        del x, k, gy, y, dx
        torch.cuda.empty_cache()
    print(f"mode {a.mode}; median ms over {a.rounds} ABAB rounds")
    print("shape".ljust(22), "path".ljust(5), *[s.rjust(12) for s in sets])
    for shape in shapes:
        for p in paths:
            vals = [sorted(res[(shape, p, s)])[len(res[(shape, p, s)]) // 2] for s in sets]
            print(" ".join(map(str, shape)).ljust(22), p.ljust(5), *[f"{v:12.4f}" for v in vals])


if __name__ == "__main__":
    main()
