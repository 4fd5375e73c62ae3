# zero-halo tap-block skipping in stencil_pad / dw_pad: parity, config 2 / 4 / 5c bench
mkdir -p gpurun_out/r62
O=gpurun_out/r62
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in config2 config4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/new_$c.json 2>&1
done
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py > $O/racecheck.log 2>&1; echo "rc=$?" >> $O/racecheck.log
