# bench with per-path CUDA graphs + L2 flush for small working sets; eager A/B
mkdir -p gpurun_out
for c in config1 config2 config3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r31_g_$c.json 2> gpurun_out/r31_g_$c.err
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-graphs > gpurun_out/r31_e_$c.json 2> gpurun_out/r31_e_$c.err
done
timeout 300 torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --config config1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r31_tr1.json 2> gpurun_out/r31_tr1.err
