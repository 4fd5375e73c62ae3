# fused backward (dX + dW in one pass): parity + a quick timing through run_shape-style calls
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x -k "fused_backward" > gpurun_out/r32_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r32_pytest.log
timeout 600 python - > gpurun_out/r32_timing.txt 2>&1 <<'PY'
import torch, paper_2604_25422_b200 as ks
for (B,H,L,K) in [(256,512,8192,7),(512,1024,16384,16)]:
    if B*H*L*4*5 > 170e9: B //= 2
    x,k,gy = ks.make_inputs(1,B,H,L,K)
    ws = torch.empty(ks.workspace_bytes(B,H,L,K,ks.HIERARCHICAL)//4+1, device="cuda")
    dx = torch.empty_like(gy); dk = torch.empty((H,K),device="cuda")
    def split():
        ks.backward_input(gy,k,ks.FUSED,out=dx); ks.backward_weight(gy,x,K,ks.HIERARCHICAL,0,ks.FUSED,out=dk,workspace=ws)
    def fused():
        ks.backward(gy,x,k,ks.FUSED,out=(dx,dk),workspace=ws)
    for name,fn in (("split",split),("fused",fused)):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        s.record(); 
        for _ in range(10): fn()
        e.record(); torch.cuda.synchronize()
        ms=s.elapsed_time(e)/10
        print(B,H,L,K,name,round(ms,4),"ms", "actual GB/s (fused 12B/elem, split 16B/elem)", round((12 if name=="fused" else 16)*B*H*L/ms/1e6,1))
    del x,gy,dx
    torch.cuda.empty_cache()
PY
