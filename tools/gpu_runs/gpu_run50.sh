# bwd_short over the 128-byte padded row view: parity suite, A/B on config 3 and 5a, ncu capture
mkdir -p gpurun_out/r50
O=gpurun_out/r50
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in config3 config5a; do
  KS_BWDS=0 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/old_$c.json 2>&1
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/new_$c.json 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_short -s 1 -c 1 -o $O/bwd5a python tools/run_shape.py 128 1024 16384 16 --reps 1 --bwd > $O/ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_short -s 1 -c 1 -o $O/bwd3 python tools/run_shape.py 256 512 8192 7 --reps 1 --bwd > $O/ncu3.log 2>&1
