mkdir -p gpurun_out
for rep in 1 2; do
for mb in 16 32 64 128; do
KS_HOST_BLOCK_MB=$mb timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/r47_mb${mb}_$rep.json 2> gpurun_out/r47_mb${mb}_$rep.err
done
done
