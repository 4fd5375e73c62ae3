O=gpurun_out/p10; mkdir -p $O
python tools/dump_plans.py $O/plans.json > $O/plans.log 2>&1
for v in cur spold; do
  if [ $v = cur ]; then L=""; else L=build/variants/$v/libks_dwconv1d.so; fi
  for c in "1024 256 2048 256" "64 1024 16384 128" "64 128 4096 4096"; do
    echo "== $v" >> $O/ab.log
    KS_LIB=$L python tools/time_paths.py $c --mode fused --reps 7 --paths fwd,dx >> $O/ab.log 2>&1
  done
done
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "fwd_dx_bitwise or padded_view or non_finite or full_config_channel or concurrent or plan_is" > $O/t.log 2>&1; echo rc=$? >> $O/t.log
timeout 600 tests/cpp/test_dropin > $O/cpp.log 2>&1; echo rc=$? >> $O/cpp.log
