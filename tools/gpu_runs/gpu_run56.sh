# stage-count sweep for the padded-view compute-bound kernels now that the producer lane parks
mkdir -p gpurun_out/r56
O=gpurun_out/r56
for c in config4 config5b config2; do
  for ns in 1 2 3 4; do
    KS_PAD_NS=$ns KS_DWPAD_NS=$ns timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/${c}_ns$ns.json 2>&1
  done
done
