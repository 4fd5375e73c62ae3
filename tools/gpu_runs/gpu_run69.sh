# per-instantiation shfl / anti-diagonal choice in stencil_pad: parity + timing vs base
mkdir -p gpurun_out/r69
O=gpurun_out/r69
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do
for v in base default; do
  if [ $v = default ]; then L=""; else L=build/variants/$v/libks_dwconv1d.so; fi
  echo "== $v" >> $O/t.log
  KS_LIB=$L python tools/time_paths.py 1024 256 2048 256 --reps 6 --paths fwd,dx >> $O/t.log 2>&1
  KS_LIB=$L python tools/time_paths.py 128 1024 16384 128 --reps 4 --paths fwd,dx >> $O/t.log 2>&1
  KS_LIB=$L python tools/time_paths.py 64 128 4096 4096 --reps 6 --paths fwd,dx >> $O/t.log 2>&1
  KS_LIB=$L python tools/time_paths.py 64 1024 16384 1024 --reps 3 --paths fwd,dx >> $O/t.log 2>&1
done
done
