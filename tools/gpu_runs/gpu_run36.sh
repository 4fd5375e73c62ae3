# after the NS change: full GPU suite, smoke, bench lines for configs 3 / 5a
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/r36_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r36_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r36_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r36_smoke.log
timeout 900 python bench.py > gpurun_out/r36_bench_config3.json 2> gpurun_out/r36_bench_config3.err
timeout 600 python bench.py --config config5a --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r36_bench_config5a.json 2> gpurun_out/r36_bench_config5a.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r36_bench_reference.json 2> gpurun_out/r36_bench_reference.err
