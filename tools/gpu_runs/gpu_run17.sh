# ncu full captures of the compute-bound kernels at small-K shapes (config 4, config 5b at B=32) and the K=16 stencil (config 5a at B=64)
mkdir -p gpurun_out
rm -f gpurun_out/r17_*.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_cb|dw_cb" -s 2 -c 2 -o gpurun_out/r17_cb4 python tools/run_shape.py 256 256 2048 256 > gpurun_out/r17_1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_cb|dw_cb" -s 2 -c 2 -o gpurun_out/r17_cb5b python tools/run_shape.py 32 1024 16384 128 > gpurun_out/r17_2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_tma|dw_tma" -s 2 -c 2 -o gpurun_out/r17_tma5a python tools/run_shape.py 64 1024 16384 16 > gpurun_out/r17_3.log 2>&1
