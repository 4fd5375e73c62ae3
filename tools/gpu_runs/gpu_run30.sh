# per-thread stage release (racecheck), stencil_pad at L = 1024 (config 1), perf check
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck.log
timeout 1500 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/sanitize_synccheck.log
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r30_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r30_pytest.log
for c in config1 config4 config5b; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r30_$c.json 2>&1
done
