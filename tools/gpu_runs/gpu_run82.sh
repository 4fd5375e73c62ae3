# ncu full captures of the compute-bound kernels as they stand (CSV export on the box)
O=gpurun_out/ncu82
mkdir -p $O
cap() {  # name, kernel regex, skip, count, command...
  n=$1; k=$2; s=$3; c=$4; shift 4
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c $c -o /tmp/$n "$@" > $O/$n.log 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > $O/$n.csv 2>> $O/$n.log
}
cap pad2 "stencil_pad|dw_pad" 0 3 python tools/run_shape.py 64 128 4096 4096 --reps 1
cap pad4 "stencil_pad|dw_pad" 0 3 python tools/run_shape.py 256 256 2048 256 --reps 1
cap pad5c dw_pad 0 1 python tools/run_shape.py 16 1024 16384 1024 --reps 1
