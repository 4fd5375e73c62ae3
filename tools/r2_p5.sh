O=gpurun_out/p5; mkdir -p $O
python tools/dump_plans.py $O/plans.json > $O/plans.log 2>&1
cp $O/plans.json profiles/r02_plans.json
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "fwd_dx_bitwise or padded_view or full_config_channel or unaligned or plan_is_current or mode_independent" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
for c in "64 128 4096 4096" "4 128 4096 4096" "16 64 1024 64" "64 1024 4096 2048"; do
  python tools/time_paths.py $c --mode fused --reps 5 --paths fwd,dx >> $O/time.log 2>&1
done
tail -3 $O/tests.log
