O=gpurun_out/p8; mkdir -p $O
for c in "1024 256 2048 256" "64 1024 16384 128" "64 128 4096 4096" "32 1024 16384 1024"; do
  python tools/time_paths.py $c --mode fused --reps 7 --paths fwd,dx >> $O/time.log 2>&1
done
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "fwd_dx_bitwise or padded_view or non_finite or full_config_channel" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
tail -2 $O/tests.log
