mkdir -p gpurun_out
for c in config5b config5c config4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dw_tma -s 1 -c 1 -o gpurun_out/prof_dw_c2 python bench.py --config config2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c2b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_tma -s 1 -c 1 -o gpurun_out/prof_stencil_c2 python bench.py --config config2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c2a.log 2>&1
