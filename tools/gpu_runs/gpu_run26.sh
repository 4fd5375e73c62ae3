# memory-bound stencil: R=16 (TMA store) vs R=32 (direct stores) at configs 3 and 5a, stage sweep
mkdir -p gpurun_out
for c in config3 config5a; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r26_base_$c.json 2>&1
  for ns in 2 3 4; do
    KS_STENCIL_R=32 KS_STENCIL_NS=$ns timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r26_r32ns${ns}_$c.json 2>&1
  done
done
