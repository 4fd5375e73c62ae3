# ncu --set full + per-launch SASS source pages of the compute-bound kernels (dw_pad at the config-4 shape, stencil_pad / dw_pad at config 2)
O=gpurun_out/ncu2; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dw_pad" -s 1 -c 1 -o $O/dw4 python tools/run_shape.py 256 256 2048 256 --reps 2 --mode fused > $O/ncu_dw4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_pad|dw_pad" -s 3 -c 3 -o $O/c2 python tools/run_shape.py 16 128 4096 4096 --reps 2 --mode fused > $O/ncu_c2.log 2>&1
for r in dw4 c2; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
  n=$(ncu -i $O/$r.ncu-rep --page raw --csv 2>/dev/null | tail -n +3 | wc -l)
  for i in $(seq 1 $n); do ncu -i $O/$r.ncu-rep --page source --csv --print-source sass --launch-skip $((i-1)) --launch-count 1 > $O/${r}_src_$i.csv 2>/dev/null; done
  rm -f $O/$r.ncu-rep
done
ls -la $O
