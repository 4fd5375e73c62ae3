# A/B library variants for the short-kernel stencil/backward: evict_first hints, stage counts
mkdir -p gpurun_out/r63
O=gpurun_out/r63
for i in 1 2; do
for v in default ef ns6 ns3m5; do
  if [ $v = default ]; then L=""; else L=build/variants/$v/libks_dwconv1d.so; fi
  echo "== $v" >> $O/t.log
  KS_LIB=$L python tools/time_paths.py 256 512 8192 7 --reps 8 >> $O/t.log 2>&1
  KS_LIB=$L python tools/time_paths.py 256 512 8192 16 --reps 8 --paths fwd,bwd >> $O/t.log 2>&1
done
done
