# stencil_tma tuning at config 5a (K = 16): threads per CTA x stages
mkdir -p gpurun_out
for nt in 128 256; do
  for ns in 2 3 4; do
    KS_STENCIL_NT=$nt KS_STENCIL_NS=$ns timeout 600 python bench.py --config config5a --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --bwd split > gpurun_out/r43_nt${nt}_ns${ns}.json 2>&1
  done
done
