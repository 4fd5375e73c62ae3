#!/usr/bin/env python3
"""Markdown results table from the committed bench lines
(profiles/r02_bench_<config>_<mode>.json, written by tools/collect_evidence.sh):
per config and mode the per-path times with their roof fraction (HBM-bound
paths: TB/s of the path's bytes; FP32-bound: fraction of the FP32 roof on
useful FLOPs, halved for a Separate-mode stencil) and the step time.

usage: python tools/results_table.py [profiles]
"""
import json
import os
import sys

P = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                         "profiles")
CONFIGS = ["config1", "config2", "config3", "config4", "config5a", "config5b", "config5c"]


def cell(p):
    if p is None:
        return "-"
    ms = p["ms"]
    t = f"{ms * 1000:.1f} µs" if ms < 0.1 else f"{ms:.2f} ms"
    if "frac_fp32_roof" in p:
        return f"{t}, {100 * p['frac_fp32_roof']:.0f}%"
    return f"{t}, {p['GB_s'] / 1000:.2f} TB/s"


def main():
    print("| config | mode | fwd | dX | dW | step (fwd + bwd) |")
    print("|---|---|---|---|---|---|")
    for c in CONFIGS:
        for m in ("separate", "fused"):
            f = os.path.join(P, f"r02_bench_{c}_{m}.json")
            if not os.path.exists(f):
                continue
            try:
                d = json.loads(open(f).read().strip().splitlines()[-1])
            except (ValueError, IndexError):
                continue
            ps = d.get("paths", {})
            step = d["ms_per_step"]
            st = f"{step * 1000:.1f} µs" if step < 0.1 else f"{step:.2f} ms"
            cfg = d.get("config", {})
            shape = f"({cfg.get('B')},{cfg.get('H')},{cfg.get('L')},{cfg.get('K')})"
            print(f"| {c[6:]} {shape} | {m} | {cell(ps.get('fwd'))} | {cell(ps.get('dX'))} | {cell(ps.get('dW'))} | {st} |")


if __name__ == "__main__":
    main()
