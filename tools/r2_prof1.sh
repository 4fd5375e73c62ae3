# plans, per-path timings in both modes, ncu --set full of the separate-mode fused backward at config 3
mkdir -p gpurun_out/p1
O=gpurun_out/p1
python tools/dump_plans.py $O/plans.json > $O/plans.log 2>&1
python tools/b200_device_spec.py $O/b200_device_spec.json > $O/spec.log 2>&1
for m in separate fused; do python tools/time_paths.py 256 512 8192 7 --mode $m --reps 20 >> $O/time_c3.log 2>&1; done
python tools/time_paths.py 512 1024 16384 16 --mode separate --reps 5 >> $O/time_c5a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd_short -s 2 -c 2 -o $O/bwd7 python tools/run_shape.py 256 512 8192 7 --reps 2 --bwd > $O/ncu_bwd7.log 2>&1
ncu -i $O/bwd7.ncu-rep --page raw --csv > $O/bwd7_raw.csv 2>/dev/null
ncu -i $O/bwd7.ncu-rep --page source --csv --print-source sass > $O/bwd7_src.csv 2>/dev/null
ls -la $O
