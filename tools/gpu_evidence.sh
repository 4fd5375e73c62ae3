# Refresh the committed evidence for the current kernels (one GPU; never multi-rank under ncu).
mkdir -p gpurun_out
rm -f gpurun_out/ev_*.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_tma -s 1 -c 1 -o gpurun_out/ev_stencil python tools/run_shape.py 256 512 8192 7 > gpurun_out/ev1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dw_tma -s 1 -c 1 -o gpurun_out/ev_dw python tools/run_shape.py 256 512 8192 7 > gpurun_out/ev2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dw_pairwise_tma -s 1 -c 1 -o gpurun_out/ev_pairwise python tools/run_shape.py 256 512 8192 7 --scheme pairwise > gpurun_out/ev3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_cb|dw_cb" -s 2 -c 2 -o gpurun_out/ev_cb python tools/run_shape.py 64 128 4096 4096 > gpurun_out/ev4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_rows|dw_rows" -s 2 -c 2 -o gpurun_out/ev_rows python tools/run_shape.py 16384 128 48 48 > gpurun_out/ev5.log 2>&1
