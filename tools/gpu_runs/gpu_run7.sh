mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in config2 config4 config5b; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python bench.py --config config3 --scheme pairwise --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_config3_pw.json 2> gpurun_out/bench_config3_pw.err
