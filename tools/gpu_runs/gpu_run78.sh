# e2e host-step block size sweep (KS_HOST_BLOCK_MB), config 3
mkdir -p gpurun_out/r78
O=gpurun_out/r78
for mb in 16 32 64 128 256 512; do
  KS_HOST_BLOCK_MB=$mb timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 4 > $O/mb$mb.json 2>&1
done
