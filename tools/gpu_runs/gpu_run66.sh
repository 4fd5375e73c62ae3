# Evidence refresh, part 2: ncu full captures exported to raw CSV on the box (reports are too big to bring back)
O=gpurun_out/ncu66
mkdir -p $O
cap() {  # name, kernel regex, skip, count, command...
  n=$1; k=$2; s=$3; c=$4; shift 4
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $s -c $c -o /tmp/$n "$@" > $O/$n.log 2>&1
  ncu -i /tmp/$n.ncu-rep --page raw --csv > $O/$n.csv 2>> $O/$n.log
  ncu -i /tmp/$n.ncu-rep --page details --csv > $O/${n}_details.csv 2>> $O/$n.log
}
cap short3 bwd_short 0 4 python tools/run_shape.py 256 512 8192 7 --reps 1 --bwd
cap short5a bwd_short 3 1 python tools/run_shape.py 128 1024 16384 16 --reps 1 --bwd
cap pad2 "stencil_pad|dw_pad" 0 3 python tools/run_shape.py 64 128 4096 4096 --reps 1
cap pad5b stencil_pad 0 1 python tools/run_shape.py 128 1024 16384 128 --reps 1
