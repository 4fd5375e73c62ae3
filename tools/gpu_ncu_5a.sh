# ncu full captures: fused backward at config 5a (K=16), stencil_pad fwd at config 5b (K=128)
mkdir -p gpurun_out/ncu5
O=gpurun_out/ncu5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dw_tma -s 1 -c 1 -o $O/bwd5a python tools/run_shape.py 128 1024 16384 16 --reps 1 --bwd > $O/bwd5a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_pad -c 1 -o $O/pad5b python tools/run_shape.py 128 1024 16384 128 --reps 1 > $O/pad5b.log 2>&1
