#!/usr/bin/env python3
"""Step-structure diagnostics at config 3 (not a bench line): the fwd +
backward step replayed as two CUDA graphs, as one graph, and eagerly, in
both orders, with the per-kernel CUDA-event split -- to see how much of the
step is gaps between launches."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2604_25422_b200 as ks

B, H, L, K = 256, 512, 8192, 7
x, k, gy = ks.make_inputs(1, B, H, L, K)
y = torch.empty_like(x); dx = torch.empty_like(gy); dk = torch.empty((H, K), device='cuda')
ws = torch.empty(ks.workspace_bytes(B, H, L, K, ks.HIERARCHICAL) // 4 + 1, device='cuda')
m = ks.SEPARATE
def fwd(): ks.forward(x, k, m, out=y)
def bwd(): ks.backward(gy, x, k, m, out=(dx, dk), workspace=ws)
def step(): fwd(); bwd()
for _ in range(5): step()
torch.cuda.synchronize()

def t(fn, n=30):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    for _ in range(5): fn()
    torch.cuda.synchronize(); s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / n

gf = torch.cuda.CUDAGraph()
with torch.cuda.graph(gf): fwd()
gb = torch.cuda.CUDAGraph()
with torch.cuda.graph(gb): bwd()
g1 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g1): step()
for rep in range(2):
    print('eager step', round(t(step), 4), ' two graphs', round(t(lambda: (gf.replay(), gb.replay())), 4),
          ' one graph', round(t(g1.replay), 4))
    print('  fwd graph alone', round(t(gf.replay), 4), ' bwd graph alone', round(t(gb.replay), 4),
          ' eager fwd', round(t(fwd), 4), ' eager bwd', round(t(bwd), 4))
# events around each path inside a replayed step
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tot = [0.0, 0.0]
for i in range(30):
    ev[0].record(); gf.replay(); ev[1].record(); gb.replay(); ev[2].record()
torch.cuda.synchronize()
print('last step split fwd', ev[0].elapsed_time(ev[1]), 'bwd', ev[1].elapsed_time(ev[2]))
