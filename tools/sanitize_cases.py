"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck).

usage (GPU box):
  compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
  compute-sanitizer --tool racecheck python tools/sanitize_cases.py
Covers the TMA paths (L % 32 == 0), the generic fallbacks (ragged L), every
dW scheme and both multiply-add modes, and checks results against the oracle
so a sanitizer-clean run is also a correct run.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_25422_b200 as ks  # noqa: E402
from oracle.oracle import CHUNKED, PAIRWISE, SEQUENTIAL, Oracle  # noqa: E402

o = Oracle()
shapes = [(2, 3, 4096, 7), (2, 2, 1024, 64), (1, 2, 2048, 256), (2, 2, 1000, 5), (1, 1, 96, 40),
          (2, 3, 4095, 7), (1, 2, 1023, 40)]  # odd L: the generic kernels' shifted aligned loads
for (B, H, L, K) in shapes:
    x, k, gy = o.fill_inputs(3, B, H, L, K)
    dx_, dk_, dgy = (torch.from_numpy(a).cuda() for a in (x, k, gy))
    for mode in (0, 1):
        y = ks.forward(dx_, dk_, mode)
        d = ks.backward_input(dgy, dk_, mode)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), o.forward(x, k, mode))
        assert np.array_equal(d.cpu().numpy(), o.backward_input(gy, k, mode))
        for s, c in ((ks.HIERARCHICAL, 0), (PAIRWISE, 0), (CHUNKED, 300), (SEQUENTIAL, 0)):
            if s == SEQUENTIAL and B * L > 5000:
                continue
            dk = ks.backward_weight(dgy, dx_, K, s, c, mode)
            torch.cuda.synchronize()
            if s != ks.HIERARCHICAL:
                assert np.array_equal(dk.cpu().numpy(), o.backward_weight(gy, x, K, s, c, mode))
    yh, dxh, dkh = ks.step_host(x, k, gy, scheme=ks.HIERARCHICAL, mode=1)

# the padded-TMA-view kernels (stencil_pad, dw_pad) with several tiles / work
# items per CTA, so every stage ring slot and both mbarrier phases recur:
# (32,64,2048,64) -> 1024 fwd/dX tiles over <= 444 CTAs; (32,256,2048,128) ->
# 4 dW work items per CTA (> NS = 3 stages); odd p (K = 150) shifts the tap origin
# (64,32,4096,7): fused backward (dX + dW in one pass), several work items per CTA
# (2400,16,48,48): short-row chunks reused round the stage ring (paper shape rows)
# (40,16,2080,16), (8,4,4160,13): K-specialised short-kernel stencils (persistent,
# more rows than CTAs), dW and fused backward with ragged last tiles
# (2,4,4096,4096), (3,8,1024,1024): K comparable to L -> stencil_pad's mirrored,
# rotating lane rings with per-lane zero-halo bounds
# (40,2,2048,1030), (32,3,1024,700): K comparable to L with >= 32 batch rows ->
# the batch-lane stencil (piece ring wraps several times, ragged row group, S = 1..3)
# (37,6,256,7), (13,3,1024,12): K <= 16 dW on rows shorter than an item -> items of
# whole rows (ragged last item); (24,8,256,32): short rows through stencil_ldg's
# whole-row CTAs; (20,4,2048,24), (9,3,512,20), (6,4,4096,28): bwd_short dW and
# stencils for 16 < K <= 32
for (B, H, L, K) in [(32, 64, 2048, 64), (32, 256, 2048, 128), (4, 8, 4096, 150), (64, 32, 4096, 7), (2400, 16, 48, 48),
                     (40, 16, 2080, 16), (8, 4, 4160, 13), (2, 4, 4096, 4096), (3, 8, 1024, 1024),
                     (40, 2, 2048, 1030), (32, 3, 1024, 700), (37, 6, 256, 7), (13, 3, 1024, 12), (24, 8, 256, 32),
                     (20, 4, 2048, 24), (9, 3, 512, 20), (6, 4, 4096, 28)]:
    x, k, gy = o.fill_inputs(5, B, H, L, K)
    dx_, dk_, dgy = (torch.from_numpy(a).cuda() for a in (x, k, gy))
    y = ks.forward(dx_, dk_, 1)
    d = ks.backward_input(dgy, dk_, 1)
    dk = ks.backward_weight(dgy, dx_, K, ks.HIERARCHICAL, 0, 1)
    if L % 32 == 0 and L >= 2048 and K <= 16:
        ks.backward(dgy, dx_, dk_, 1)
    torch.cuda.synchronize()
    xs = np.ascontiguousarray(x[:, :1])
    gs = np.ascontiguousarray(gy[:, :1])
    kk = np.ascontiguousarray(k[:1])
    assert np.array_equal(y.cpu().numpy()[:, :1], o.forward(xs, kk, 1))
    assert np.array_equal(d.cpu().numpy()[:, :1], o.backward_input(gs, kk, 1))
    truth = o.backward_weight(gs.astype(np.float64), xs.astype(np.float64), K, SEQUENTIAL)
    err = np.abs(dk.cpu().numpy()[:1] - truth).max() / np.abs(truth).max()
    assert err <= 1e-4, err
# unaligned bases: HIERARCHICAL dW stages the inputs into aligned scratch
x, k, gy = o.fill_inputs(9, 3, 4, 2048, 16)
buf = torch.empty(2 * x.size + 8, device="cuda")
xs_ = buf[1:1 + x.size].view(x.shape)
gs_ = buf[x.size + 5:x.size + 5 + x.size].view(x.shape)
xs_.copy_(torch.from_numpy(x))
gs_.copy_(torch.from_numpy(gy))
a = ks.backward_weight(gs_, xs_, 16, ks.HIERARCHICAL, 0, 1)
b = ks.backward_weight(torch.from_numpy(gy).cuda(), torch.from_numpy(x).cuda(), 16, ks.HIERARCHICAL, 0, 1)
torch.cuda.synchronize()
assert torch.equal(a.view(torch.int32), b.view(torch.int32))
print("sanitize cases ok")
