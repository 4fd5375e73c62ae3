# refresh the committed evidence for the padded-view kernels + every bench line
mkdir -p gpurun_out
rm -f gpurun_out/r25_*.ncu-rep
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/r25_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r25_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r25_bench_config3.json 2> gpurun_out/r25_bench_config3.err
for c in config1 config2 config4 config5a config5b; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r25_bench_$c.json 2> gpurun_out/r25_bench_$c.err
done
timeout 900 python bench.py --config config5c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r25_bench_config5c.json 2> gpurun_out/r25_bench_config5c.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_pad|dw_pad" -s 2 -c 3 -o gpurun_out/r25_pad4 python tools/run_shape.py 256 256 2048 256 > gpurun_out/r25_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_pad|dw_pad" -s 2 -c 3 -o gpurun_out/r25_pad2 python tools/run_shape.py 16 128 4096 4096 > gpurun_out/r25_ncu2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/r25_launches4.csv python bench.py --config config4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r25_launches4.log 2>&1
