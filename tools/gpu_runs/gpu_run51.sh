# K-specialised stencils: parity suite, A/B (KS_STS=0 = stencil_tma) on config 3 and 5a, ncu of the config-3 forward
mkdir -p gpurun_out/r51
O=gpurun_out/r51
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for c in config3 config5a; do
  KS_STS=0 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/old_$c.json 2>&1
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/new_$c.json 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_short -c 1 -o $O/st3 python tools/run_shape.py 256 512 8192 7 --reps 1 > $O/ncu3.log 2>&1
