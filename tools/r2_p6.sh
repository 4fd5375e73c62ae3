O=gpurun_out/p6; mkdir -p $O
for c in "64 128 4096 4096" "16 64 1024 64" "64 1024 4096 2048" "1024 256 2048 256"; do
  python tools/time_paths.py $c --mode fused --reps 5 --paths fwd,dx >> $O/time.log 2>&1
done
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "fwd_dx_bitwise or padded_view or full_config_channel or non_finite" > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
tail -2 $O/tests.log
