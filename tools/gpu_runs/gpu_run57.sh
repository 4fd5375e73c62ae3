# copy vs stencil headroom at config 3 shapes
mkdir -p gpurun_out/r57
O=gpurun_out/r57
for K in 1 7 16; do python tools/time_paths.py 256 512 8192 $K --reps 10 >> $O/t.log 2>&1; done
KS_STS=0 python tools/time_paths.py 256 512 8192 7 --reps 10 --paths fwd,dx >> $O/t.log 2>&1
