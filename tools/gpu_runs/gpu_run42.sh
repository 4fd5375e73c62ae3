# checkpoint: full GPU suite, smoke, sanitizers (incl. fused backward + short-row multi-chunk), default bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/r42_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r42_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r42_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r42_smoke.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
timeout 900 python bench.py > gpurun_out/r42_bench_config3.json 2> gpurun_out/r42_bench_config3.err
