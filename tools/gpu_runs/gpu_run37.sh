# ncu of the fused backward and the forward at config 5a's shape (B = 64)
mkdir -p gpurun_out
rm -f gpurun_out/r37_*.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dw_tma|stencil_tma" -s 2 -c 2 -o gpurun_out/r37_5a python -c "
import torch, paper_2604_25422_b200 as ks
B,H,L,K=64,1024,16384,16
x,k,gy=ks.make_inputs(1,B,H,L,K)
for _ in range(2):
    ks.forward(x,k,ks.FUSED); ks.backward(gy,x,k,ks.FUSED)
torch.cuda.synchronize()" > gpurun_out/r37_ncu.log 2>&1
