mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_rows|dw_rows" -s 2 -c 2 -o gpurun_out/prof_rows python tools/run_shape.py 16384 128 48 48 > gpurun_out/ncu_rows.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"stencil_cb" -s 1 -c 1 -o gpurun_out/prof_cb_c4 python tools/run_shape.py 1024 256 2048 256 > gpurun_out/ncu_cb.log 2>&1
