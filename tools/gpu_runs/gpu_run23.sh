# padded-view kernels final: full GPU suite, smoke, every config's bench line, NS sweep for long K
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/r23_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r23_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r23_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r23_smoke.log
for c in config1 config2 config4 config5b; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r23_bench_$c.json 2> gpurun_out/r23_bench_$c.err
done
KS_PAD_NS=2 timeout 600 python bench.py --config config2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r23_ns2_config2.json 2> gpurun_out/r23_ns2_config2.err
timeout 900 python bench.py --config config5c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r23_bench_config5c.json 2> gpurun_out/r23_bench_config5c.err
KS_PAD_NS=2 timeout 900 python bench.py --config config5c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r23_ns2_config5c.json 2> gpurun_out/r23_ns2_config5c.err
