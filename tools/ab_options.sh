# usage: bash tools/ab_options.sh TAG "B H L K" fwd,dx - opt=v,opt2=w ...   (on the GPU box, via gpurun)
# option sweep at one shape: $1 tag, $2 shape, $3 paths, then option sets (each "a=1,b=2"; "-" = defaults)
O=gpurun_out/ab_$1; mkdir -p $O; SH=$2; P=$3; shift 3
for rep in 1 2 3; do
  for o in "$@"; do
    OPT=""; if [ "$o" != "-" ]; then for kv in ${o//,/ }; do OPT="$OPT --opt $kv"; done; fi
    echo "== $o rep$rep" >> $O/ab.log
    timeout 300 python tools/time_paths.py $SH --mode fused --reps 5 --paths $P $OPT >> $O/ab.log 2>&1
  done
done
python tools/ab_table.py $O/ab.log
