O=gpurun_out/p9; mkdir -p $O
for rep in 1 2; do
for v in cur spold; do
  if [ $v = cur ]; then L=""; else L=build/variants/$v/libks_dwconv1d.so; fi
  for c in "1024 256 2048 256" "64 1024 16384 128"; do
    echo "== $v rep$rep" >> $O/ab.log
    KS_LIB=$L python tools/time_paths.py $c --mode fused --reps 7 --paths fwd,dx >> $O/ab.log 2>&1
  done
done
done
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "concurrent" > $O/t.log 2>&1; echo rc=$? >> $O/t.log
timeout 600 tests/cpp/test_dropin > $O/cpp.log 2>&1; echo rc=$? >> $O/cpp.log
tail -3 $O/t.log $O/cpp.log
