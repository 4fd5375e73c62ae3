# direct-store vs TMA-store sweep over K for the short-kernel stencils (config 3 and 5a rows)
mkdir -p gpurun_out/r59
O=gpurun_out/r59
for K in 3 5 7 8 9 11 13 16; do
  for d in 0 1; do KS_DST=$d python tools/time_paths.py 256 512 8192 $K --reps 8 --paths fwd,dx >> $O/t3.log 2>&1; done
done
for K in 7 16; do
  for d in 0 1; do KS_DST=$d python tools/time_paths.py 64 1024 16384 $K --reps 8 --paths fwd,dx,bwd >> $O/t5.log 2>&1; done
done
