#!/bin/bash
# A/B of the working tree's library against build/variants/old (a build of HEAD's csrc:
#   tools/build_variant.sh old "" <HEAD csrc>), graph-timed, over shapes $1 (;-separated),
#   paths $2, in both modes; output in gpurun_out/ab_head_$3/.
O=gpurun_out/ab_head_$3; mkdir -p $O
for m in separate fused; do
  for v in old cur; do
    L=""; [ $v = old ] && L=build/variants/old/libks_dwconv1d.so
    echo "== $v" >> $O/$m.txt
    KS_LIB=$L timeout 600 python tools/sweep_options.py --graph --inner 5 --shapes "$1" --sets=- --paths $2 --mode $m --reps 5 >> $O/$m.txt 2>&1
  done
done
