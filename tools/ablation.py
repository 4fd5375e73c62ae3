#!/usr/bin/env python3
"""The paper's kernel ablation (Table II) re-run on B200.

usage: python tools/ablation.py [--shape B H L K] [--reps N] [--mode separate|fused] [--out profiles/r02_ablation]

Times forward / dX / dW of the four paper designs (naive, coalesced, shared,
warp; csrc/paper_variants.cu, the reference's launch geometries) and of this
library's kernels (variant b200) on the paper's training shape (B,H,L,K) =
(16384,128,48,48) by default, with CUDA events after warm-up.  Writes, in the
reference's timing-log schema (variant,path,runtime_ms,run_id;
src/timing_log.cpp:44-97), which the reference's own analysis pipeline reads
(oracle/_ref/ks_b200_report, with a B200 device spec):
  <out>_paper.csv    the paper's designs that launch all three paths here;
  <out>_library.csv  the paper's naive design (the baseline) and this library,
                     logged under the warp-tiled id -- the design family it
                     extends; the reference's VariantId has no fifth value;
and <out>.md with the table and per-path effective bandwidth.
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_25422_b200 as ks  # noqa: E402


def time_it(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", type=int, nargs=4, default=[16384, 128, 48, 48])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="profiles/r02_ablation")
    ap.add_argument("--mode", choices=["separate", "fused"], default="separate")
    a = ap.parse_args()
    B, H, L, K = a.shape
    mode = ks.FUSED if a.mode == "fused" else ks.SEPARATE
    x, k, gy = ks.make_inputs(1, B, H, L, K)
    y = torch.empty_like(x)
    dk = torch.empty((H, K), dtype=torch.float32, device="cuda")
    ws = torch.empty(max(1, ks.workspace_bytes(B, H, L, K, ks.HIERARCHICAL) // 4), device="cuda")
    rows, table = [], []
    path_bytes = 8 * B * H * L + 4 * H * K
    for name in ("naive", "coalesced", "shared", "warp", "b200"):
        res = {}
        for path in ("fwd", "dx", "dw"):
            if name == "b200":
                fn = {"fwd": lambda: ks.forward(x, k, mode, out=y),
                      "dx": lambda: ks.backward_input(gy, k, mode, out=y),
                      "dw": lambda: ks.backward_weight(gy, x, K, ks.HIERARCHICAL, 0, mode, out=dk,
                                                       workspace=ws)}[path]
            else:
                fn = {"fwd": lambda: ks.variant(name, "fwd", x, k, mode=mode, out=y),
                      "dx": lambda: ks.variant(name, "dx", gy, k, mode=mode, out=y),
                      "dw": lambda: ks.variant(name, "dw", gy, x, K, mode=mode, out=dk)}[path]
            try:
                ts = time_it(fn, a.reps)
            except ks.KsError as err:
                res[path] = None
                print(f"{name} {path}: not launchable at this shape ({err})")
                continue
            res[path] = sorted(ts)[len(ts) // 2]
            ref_path = {"fwd": "fwd", "dx": "bwd_in", "dw": "bwd_k"}[path]
            rows.append((name, [f"{ref_path},{t:.6f},{i}" for i, t in enumerate(ts)]))
        total = sum(res.values()) if all(v is not None for v in res.values()) else None
        table.append((name, res, total))
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    complete = {name for name, _, total in table if total is not None}
    head = f"shape (B,H,L,K)=({B},{H},{L},{K}), fp32 {a.mode}, {a.reps} CUDA-event timings per path on one B200"
    with open(a.out + "_paper.csv", "w") as f:
        f.write(f"# the paper's kernel designs as sm_100a kernels (csrc/paper_variants.cu), {head}; "
                f"designs that cannot launch every path at this shape are left out\n")
        f.write("variant,path,runtime_ms,run_id\n")
        for name, rs in rows:
            if name != "b200" and name in complete:
                f.write("".join(f"{name},{r}\n" for r in rs))
    with open(a.out + "_library.csv", "w") as f:
        f.write(f"# naive = the paper's naive design; warp = THIS LIBRARY's kernels (the warp-tiled design "
                f"family it extends; the reference's VariantId has no fifth value), {head}\n")
        f.write("variant,path,runtime_ms,run_id\n")
        for name, rs in rows:
            if name in ("naive", "b200"):
                f.write("".join(f"{'warp' if name == 'b200' else name},{r}\n" for r in rs))
    naive_total = table[0][2]
    with open(a.out + ".md", "w") as f:
        f.write(f"# Paper ablation on one B200 — (B,H,L,K) = ({B},{H},{L},{K}), fp32, {a.mode}\n\n")
        f.write("Median of %d CUDA-event timings after 3 warm-ups (ms); GB/s = (8·B·H·L + 4·H·K) / time.\n\n" % a.reps)
        f.write("| variant | fwd ms | dX ms | dW ms | conv total ms | speedup vs naive | fwd GB/s | dX GB/s | dW GB/s |\n")
        f.write("|---|---|---|---|---|---|---|---|---|\n")
        for name, res, total in table:
            cell = lambda v: f"{v:.3f}" if v is not None else "n/a"  # noqa: E731
            gbs = lambda v: f"{path_bytes / v / 1e6:.0f}" if v else "n/a"  # noqa: E731
            sp = f"{naive_total / total:.2f}x" if (total and naive_total) else "n/a"
            f.write(f"| {name} | {cell(res.get('fwd'))} | {cell(res.get('dx'))} | {cell(res.get('dw'))} | "
                    f"{cell(total)} | {sp} | {gbs(res.get('fwd'))} | {gbs(res.get('dx'))} | {gbs(res.get('dw'))} |\n")
        f.write("\nPaper (Tesla P100, same shape, PAPER.md:565-568): naive 29.97 / 30.25 / 73.26 = 133.47 ms; "
                "coalesced 106.65; shared 66.57; warp 10.46 / 10.61 / 19.91 = 40.99 ms.\n")
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    main()
