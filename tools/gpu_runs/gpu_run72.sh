# stencil_pad with a provably warp-uniform tap-block range (tw broadcast): current default vs previous vs forced variants
mkdir -p gpurun_out/r72
O=gpurun_out/r72
for i in 1 2; do
for v in prev default sa s1a0; do
  if [ $v = default ]; then L=""; else L=build/variants/$v/libks_dwconv1d.so; fi
  echo "== $v" >> $O/t.log
  KS_LIB=$L python tools/time_paths.py 1024 256 2048 256 --reps 6 --paths fwd,dx >> $O/t.log 2>&1
  KS_LIB=$L python tools/time_paths.py 128 1024 16384 128 --reps 4 --paths fwd,dx >> $O/t.log 2>&1
  KS_LIB=$L python tools/time_paths.py 64 128 4096 4096 --reps 6 --paths fwd,dx >> $O/t.log 2>&1
  KS_LIB=$L python tools/time_paths.py 64 1024 16384 1024 --reps 3 --paths fwd,dx >> $O/t.log 2>&1
done
done
