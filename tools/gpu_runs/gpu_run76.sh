# fused-backward stage count for K <= 8 (4 = 2 CTAs/SM, 3 = 3 CTAs/SM, 2): config 3
mkdir -p gpurun_out/r76
O=gpurun_out/r76
for i in 1 2; do for v in default fns3 fns2; do
  if [ $v = default ]; then L=""; else L=build/variants/$v/libks_dwconv1d.so; fi
  echo "== $v" >> $O/t.log
  KS_LIB=$L python tools/time_paths.py 256 512 8192 7 --reps 8 --paths bwd >> $O/t.log 2>&1
done; done
