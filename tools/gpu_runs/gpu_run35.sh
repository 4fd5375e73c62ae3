# full launch list of the config-3 bench (split + fused loops); fused-bwd stage-count sweep at configs 3 / 5a
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 250 --csv --log-file gpurun_out/r35_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r35_launches.log 2>&1
for ns in 2 3 4; do
  for c in config3 config5a; do
    KS_DWTMA_NS=$ns timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r35_ns${ns}_$c.json 2>&1
  done
done
