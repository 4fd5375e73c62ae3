# Evidence refresh after the K-specialised short kernels: final bench/tests, sanitizers, ncu full captures
bash tools/gpu_final.sh
bash tools/gpu_sanitize.sh
O=gpurun_out/final
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_short -c 4 -o $O/short3 python tools/run_shape.py 256 512 8192 7 --reps 1 --bwd > $O/ncu_short3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_short -s 3 -c 1 -o $O/short5a python tools/run_shape.py 128 1024 16384 16 --reps 1 --bwd > $O/ncu_short5a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_pad -c 1 -o $O/pad5b python tools/run_shape.py 128 1024 16384 128 --reps 1 > $O/ncu_pad5b.log 2>&1
