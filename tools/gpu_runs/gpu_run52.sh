# padded view from 128-byte rows (4-D box {36,n,...}): parity suite, compute-bound configs
mkdir -p gpurun_out/r52
O=gpurun_out/r52
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in config2 config4 config5b; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/new_$c.json 2>&1
done
