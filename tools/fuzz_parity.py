#!/usr/bin/env python3
"""Randomised parity sweep on the GPU (not part of the test suite: minutes).

For N random shapes (B, H, L, K) -- L drawn to hit every dispatch tier
(short rows, L % 8 / % 32 / ragged, long rows) and K from 1 to 600 -- checks
fwd / dX bitwise against the oracle on sampled channels in both multiply-add
modes, dW HIERARCHICAL against the fp64 oracle to the parity tolerance, and
the fused backward bitwise against the separate calls; for small reductions
also the reference's SEQUENTIAL / PAIRWISE / CHUNKED(c) dW bit for bit.  Prints one line per
failure and a summary.

usage: python tools/fuzz_parity.py [--n 200] [--seed 0]
"""
import argparse
import os
import random
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_25422_b200 as ks  # noqa: E402
from oracle.oracle import CHUNKED, FUSED, PAIRWISE, SEPARATE, SEQUENTIAL, Oracle, normwise  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200)
ap.add_argument("--seed", type=int, default=0)
a = ap.parse_args()
rng = random.Random(a.seed)
o = Oracle()
fails = 0
for it in range(a.n):
    tier = rng.choice(["short", "l8", "l32", "ragged", "long"])
    L = {"short": rng.randint(8, 1000), "l8": 8 * rng.randint(128, 1200), "l32": 32 * rng.randint(32, 300),
         "ragged": rng.randint(1024, 9000), "long": 2048 * rng.randint(1, 8)}[tier]
    K = rng.choice([rng.randint(1, 16), rng.randint(17, 64), rng.randint(65, 600)])
    B, H = rng.randint(1, 12), rng.randint(1, 24)
    if B * H * L > 40_000_000:
        B = max(1, 40_000_000 // (H * L))
    x, k, gy = ks.make_inputs(100 + it, B, H, L, K)
    kh = k.cpu().numpy()
    hs = sorted({0, H - 1, rng.randrange(H)})
    bad = []
    for m in (SEPARATE, FUSED):
        y = ks.forward(x, k, m)
        dx = ks.backward_input(gy, k, m)
        torch.cuda.synchronize()
        for h in hs:
            xs = np.ascontiguousarray(x[:, h:h + 1].cpu().numpy())
            gs = np.ascontiguousarray(gy[:, h:h + 1].cpu().numpy())
            kk = np.ascontiguousarray(kh[h:h + 1])
            if not np.array_equal(y[:, h:h + 1].cpu().numpy().view(np.uint32), o.forward(xs, kk, m).view(np.uint32)):
                bad.append(f"fwd m={m} h={h}")
            if not np.array_equal(dx[:, h:h + 1].cpu().numpy().view(np.uint32),
                                  o.backward_input(gs, kk, m).view(np.uint32)):
                bad.append(f"dX m={m} h={h}")
    dk = ks.backward_weight(gy, x, K, ks.HIERARCHICAL, 0, FUSED)
    dx2, dk2 = ks.backward(gy, x, k, FUSED)
    dxs = ks.backward_input(gy, k, FUSED)
    torch.cuda.synchronize()
    if not torch.equal(dk.view(torch.int32), dk2.view(torch.int32)):
        bad.append("fused dk != dW call")
    if not torch.equal(dx2.view(torch.int32), dxs.view(torch.int32)):
        bad.append("fused dx != dX call")
    for h in hs:
        xs = np.ascontiguousarray(x[:, h:h + 1].cpu().numpy()).astype(np.float64)
        gs = np.ascontiguousarray(gy[:, h:h + 1].cpu().numpy()).astype(np.float64)
        truth = o.backward_weight(gs, xs, K, SEQUENTIAL)
        err = normwise(dk[h:h + 1].cpu().numpy(), truth)
        if not err <= 1e-4:
            bad.append(f"dW h={h} normwise {err:.2e}")
    # the reference's own association orders, bit for bit (small reductions only)
    if B * L <= 40000:
        h = hs[-1]
        xs = np.ascontiguousarray(x[:, h:h + 1].cpu().numpy())
        gs = np.ascontiguousarray(gy[:, h:h + 1].cpu().numpy())
        for sch, c in ((SEQUENTIAL, 0), (PAIRWISE, 0), (CHUNKED, rng.randint(1, 3000))):
            for m in (SEPARATE, FUSED):
                got = ks.backward_weight(gy, x, K, sch, c, m)[h:h + 1].cpu().numpy()
                ref = o.backward_weight(gs, xs, K, sch, c, m)
                if not np.array_equal(got.view(np.uint32), ref.view(np.uint32)):
                    bad.append(f"dW scheme={sch} chunk={c} m={m} h={h} not bitwise")
    if bad:
        fails += 1
        print(f"FAIL ({B},{H},{L},{K}) tier={tier}: {'; '.join(bad)}", flush=True)
    del x, gy, y, dx, dx2, dxs
print(f"fuzz_parity: {a.n - fails}/{a.n} shapes clean (seed {a.seed})")
sys.exit(1 if fails else 0)
