# dw_pad uniform-gy + anti-diagonal order (variant dwad) vs default: bits and timing
mkdir -p gpurun_out/r71
O=gpurun_out/r71
for s in "8 16 4096 4096" "3 4 16384 1024"; do
  n=$(echo $s | tr ' ' _)
  python tools/dw_bits.py $s /tmp/new_$n.npy > /dev/null 2>&1
  KS_LIB=build/variants/dwad/libks_dwconv1d.so python tools/dw_bits.py $s /tmp/old_$n.npy > /dev/null 2>&1
  python -c "import numpy as np; a=np.load('/tmp/new_$n.npy'); b=np.load('/tmp/old_$n.npy'); print('$n', 'bitwise equal' if (a.view(np.uint32)==b.view(np.uint32)).all() else 'DIFFER')" >> $O/bits.log 2>&1
done
for i in 1 2; do
for v in default dwad; do
  if [ $v = default ]; then L=""; else L=build/variants/$v/libks_dwconv1d.so; fi
  echo "== $v" >> $O/t.log
  KS_LIB=$L python tools/time_paths.py 64 128 4096 4096 --reps 6 --paths dw >> $O/t.log 2>&1
  KS_LIB=$L python tools/time_paths.py 64 1024 16384 1024 --reps 3 --paths dw >> $O/t.log 2>&1
done
done
