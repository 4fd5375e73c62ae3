# bwd_short with the column switch around the item math only: parity, synccheck/racecheck, config 3 / 5a
mkdir -p gpurun_out/r55
O=gpurun_out/r55
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for tool in synccheck racecheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/sanitize_$tool.log
done
for c in config3 config5a; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/new_$c.json 2>&1
done
