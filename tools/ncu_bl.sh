# ncu --set full + SASS source page of the batch-lane stencil at config 2's shape (B = 64 full batch, 16 channels)
O=gpurun_out/ncu_bl; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_bl" -s 2 -c 2 -o $O/bl python tools/run_shape.py 64 16 4096 4096 --reps 2 --mode fused > $O/ncu.log 2>&1
ncu -i $O/bl.ncu-rep --page raw --csv > $O/bl.raw.csv 2>/dev/null
for i in 1 2; do ncu -i $O/bl.ncu-rep --page source --csv --print-source sass --launch-skip $((i-1)) --launch-count 1 > $O/bl_src_$i.csv 2>/dev/null; done
rm -f $O/bl.ncu-rep
