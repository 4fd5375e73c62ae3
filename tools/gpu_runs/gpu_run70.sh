# dw_pad lanes = tap groups at NJG = 32: bitwise A/B vs the previous mapping, parity suite, timing
mkdir -p gpurun_out/r70
O=gpurun_out/r70
for s in "8 16 4096 4096" "4 8 8192 1500" "3 4 16384 1024"; do
  n=$(echo $s | tr ' ' _)
  python tools/dw_bits.py $s /tmp/new_$n.npy > /dev/null 2>&1
  KS_LIB=build/variants/nolanejg/libks_dwconv1d.so python tools/dw_bits.py $s /tmp/old_$n.npy > /dev/null 2>&1
  python -c "import numpy as np; a=np.load('/tmp/new_$n.npy'); b=np.load('/tmp/old_$n.npy'); print('$n', 'bitwise equal' if (a.view(np.uint32)==b.view(np.uint32)).all() else 'DIFFER')" >> $O/bits.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do
for v in nolanejg default; do
  if [ $v = default ]; then L=""; else L=build/variants/$v/libks_dwconv1d.so; fi
  echo "== $v" >> $O/t.log
  KS_LIB=$L python tools/time_paths.py 64 128 4096 4096 --reps 6 --paths dw >> $O/t.log 2>&1
  KS_LIB=$L python tools/time_paths.py 64 1024 16384 1024 --reps 3 --paths dw >> $O/t.log 2>&1
done
done
