# usage: [MODE=fused|separate] bash tools/ab_variants.sh "VARIANTS" TAG "B H L K;B H L K" fwd,dx,dw   (on the GPU box, via gpurun)
# A/B timing: current build vs variants "$1" (space-separated).  A variant is
#   cur                 the current build
#   NAME                build/variants/NAME (tools/build_variant.sh)
#   opt:name=val        the current build with a tuning option
#   NAME@name=val       a variant build with a tuning option
# over shapes "$3" (;-separated), paths $4, tag $2, mode $MODE (default fused)
O=gpurun_out/ab_$2; mkdir -p $O
MODE=${MODE:-fused}
IFS=';' read -ra SH <<< "$3"
for rep in 1 2 3; do
for v in cur $1; do
  L=""; OPT=""
  case $v in
    cur) ;;
    opt:*) OPT="--opt ${v#opt:}";;
    *@*) L=build/variants/${v%@*}/libks_dwconv1d.so; OPT="--opt ${v#*@}";;
    *) L=build/variants/$v/libks_dwconv1d.so;;
  esac
  for c in "${SH[@]}"; do
    echo "== $v rep$rep" >> $O/ab.log
    KS_LIB=$L timeout 300 python tools/time_paths.py $c --mode $MODE --reps 7 --paths $4 $OPT >> $O/ab.log 2>&1
  done
done
done
python tools/ab_table.py $O/ab.log
