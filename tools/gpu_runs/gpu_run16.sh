# Re-validate after container re-creation: GPU tests, smoke, default bench, every config's bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r16_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/r16_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r16_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r16_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r16_smoke.log
timeout 900 python bench.py > gpurun_out/r16_bench_config3.json 2> gpurun_out/r16_bench_config3.err
for c in config1 config2 config4 config5a config5b; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r16_bench_$c.json 2> gpurun_out/r16_bench_$c.err
done
