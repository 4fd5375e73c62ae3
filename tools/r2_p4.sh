O=gpurun_out/p4; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "fwd_dx_bitwise or padded_view or full_config_channel or unaligned or plan_is_current or mode_independent" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
python tools/dump_plans.py $O/plans.json > $O/plans.log 2>&1
for c in "64 128 4096 4096" "1024 256 2048 256" "64 1024 16384 128" "32 1024 16384 1024"; do
  python tools/time_paths.py $c --mode fused --reps 5 --paths fwd,dx >> $O/time.log 2>&1
done
python tools/time_paths.py 64 128 4096 4096 --mode fused --reps 5 --paths fwd,dx --opt pad_skip=0 >> $O/time.log 2>&1
tail -3 $O/tests.log
