# full suite + bench lines with the fused-backward step
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/r33_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r33_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r33_bench_config3.json 2> gpurun_out/r33_bench_config3.err
for c in config1 config2 config4 config5a config5b; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r33_bench_$c.json 2> gpurun_out/r33_bench_$c.err
done
timeout 600 torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r33_tr1.json 2> gpurun_out/r33_tr1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dw_tma" -s 4 -c 1 -o gpurun_out/r33_bwd3 python -c "
import torch, paper_2604_25422_b200 as ks
B,H,L,K=256,512,8192,7
x,k,gy=ks.make_inputs(1,B,H,L,K)
for _ in range(3): ks.backward(gy,x,k,ks.FUSED)
torch.cuda.synchronize()" > gpurun_out/r33_ncu.log 2>&1
