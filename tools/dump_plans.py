#!/usr/bin/env python3
"""Dump the library's launch plans (ks_dwconv1d_plan: kernel, grid, block,
dynamic smem, registers, CTAs/SM -- the real dispatch, nothing launched) for
every BASELINE config, the per-GPU shards of the multi-GPU configs and the
paper's shape, all four entry points, to JSON (the evidence the B200 traffic
model, paper_2604_25422_b200/traffic.py, is tested against on the CPU).

usage: python tools/dump_plans.py [out.json]   (needs a GPU)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_25422_b200 as ks  # noqa: E402

SHAPES = {
    "config1": (16, 64, 1024, 64), "config2": (64, 128, 4096, 4096), "config3": (256, 512, 8192, 7),
    "config4": (1024, 256, 2048, 256), "config5a": (512, 1024, 16384, 16), "config5b": (512, 1024, 16384, 128),
    "config5c": (512, 1024, 16384, 1024), "config4_g2": (512, 256, 2048, 256), "config4_g4": (256, 256, 2048, 256),
    "config4_g8": (128, 256, 2048, 256), "config5a_g8": (64, 1024, 16384, 16), "config5b_g8": (64, 1024, 16384, 128),
    "config5c_g8": (64, 1024, 16384, 1024), "paper": (16384, 128, 48, 48),
}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_plans.json"
    res = {}
    for name, (B, H, L, K) in SHAPES.items():
        res[name] = {"shape": [B, H, L, K]}
        for path in ("fwd", "dx", "dw", "bwd"):
            res[name][path] = ks.plan(path, B, H, L, K)
        res[name]["dw_pairwise"] = ks.plan("dw", B, H, L, K, scheme=ks.PAIRWISE)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(f"wrote {out}: {sum(len(v) - 1 for v in res.values())} plans")


if __name__ == "__main__":
    main()
