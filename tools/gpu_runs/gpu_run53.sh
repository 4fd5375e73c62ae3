# producer lanes park on NANOSLEEP.SYNCS (try_wait suspend hint): parity suite, compute-bound configs
mkdir -p gpurun_out/r53
O=gpurun_out/r53
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in config2 config4 config5b; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/new_$c.json 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_pad -c 1 -o $O/pad5b python tools/run_shape.py 128 1024 16384 128 --reps 1 > $O/ncu.log 2>&1
