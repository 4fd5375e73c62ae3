#!/bin/bash
# ncu --set full captures of the round-2 off-config tiers (one GPU; gpurun):
#   gpurun -- 'bash tools/ncu_offconfig.sh'  then
#   python tools/ncu_summary.py r02 --full offcfg_rows=gpurun_out/ncu_off/rows.raw.csv ...
O=gpurun_out/ncu_off; mkdir -p $O
T="timeout 600"
# short rows: stencil_ldg with whole rows per CTA (fwd), bwd_short multi-row dW items
$T ncu --set full --clock-control none --import-source on -k regex:"stencil_ldg|bwd_short" -c 3 -o $O/rows python tools/run_shape.py 8192 64 256 12 --reps 1 > $O/rows.log 2>&1
# 16 < K <= 32: bwd_short stencil (Fused, per-row) and dW with 24 accumulators
$T ncu --set full --clock-control none --import-source on -k regex:"bwd_short" -c 3 -o $O/k24 python tools/run_shape.py 128 64 16384 24 --reps 1 --mode fused > $O/k24.log 2>&1
# dw_tma multi-row items (K = 64, L = 1024)
$T ncu --set full --clock-control none --import-source on -k regex:"dw_tma" -c 1 -o $O/dwmr python tools/run_shape.py 2048 64 1024 64 --reps 1 > $O/dwmr.log 2>&1
for r in rows k24 dwmr; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
  rm -f $O/$r.ncu-rep
done
ls -la $O
