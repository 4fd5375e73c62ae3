# A/B: stencil_tma with lds4 (main) vs without (build/alt), alternating on one box
mkdir -p gpurun_out
for rep in 1 2 3; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r39_main_$rep.json 2>&1
  KS_LIB=$PWD/build/alt/libks_alt.so timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r39_alt_$rep.json 2>&1
done
