# direct stores for K >= 10 stencils: parity, 5a / 3 bench lines
mkdir -p gpurun_out/r60
O=gpurun_out/r60
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in config3 config5a; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/new_$c.json 2>&1
done
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
