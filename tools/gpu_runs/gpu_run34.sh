# evidence for the fused-backward step: launch list (config 3 default bench), ncu full of the fused kernel, bench line
mkdir -p gpurun_out
rm -f gpurun_out/r34_*.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/r34_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r34_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dw_tma" -s 1 -c 1 -o gpurun_out/r34_bwd3 python -c "
import torch, paper_2604_25422_b200 as ks
B,H,L,K=256,512,8192,7
x,k,gy=ks.make_inputs(1,B,H,L,K)
for _ in range(3): ks.backward(gy,x,k,ks.FUSED)
torch.cuda.synchronize()" > gpurun_out/r34_ncu.log 2>&1
timeout 900 python bench.py > gpurun_out/r34_bench_config3.json 2> gpurun_out/r34_bench_config3.err
