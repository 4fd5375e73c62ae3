import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_2604_25422_b200 as ks
B,H,L,K = 256,512,8192,7
x,k,gy = ks.make_inputs(1,B,H,L,K)
y=torch.empty_like(x); dx=torch.empty_like(gy); dk=torch.empty((H,K),device='cuda')
ws=torch.empty(ks.workspace_bytes(B,H,L,K,ks.HIERARCHICAL)//4+1,device='cuda')
m=ks.SEPARATE
def fwd(): ks.forward(x,k,m,out=y)
def bwd(): ks.backward(gy,x,k,m,out=(dx,dk),workspace=ws)
def step(): fwd(); bwd()
for _ in range(5): step()
torch.cuda.synchronize()
def t(fn, n=20):
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    for _ in range(3): fn()
    torch.cuda.synchronize(); s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e)/n
print('eager step', t(step))
print('eager fwd', t(fwd), 'eager bwd', t(bwd))
gf=torch.cuda.CUDAGraph()
with torch.cuda.graph(gf): fwd()
gb=torch.cuda.CUDAGraph()
with torch.cuda.graph(gb): bwd()
print('graph step', t(lambda:(gf.replay(),gb.replay())))
print('graph fwd', t(gf.replay), 'graph bwd', t(gb.replay))
g=torch.cuda.CUDAGraph()
with torch.cuda.graph(g): step()
print('one graph step', t(g.replay))
for name in ('fwd','dx','dw','bwd'):
    for r in ks.plan(name,B,H,L,K): print(name, r)
print(ks.plan('fwd',64,128,4096,4096)); print(ks.plan('dw',1024,256,2048,256)); print(ks.plan('bwd',512,1024,16384,16))
