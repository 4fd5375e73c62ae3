# stencil_ldg at K = 16: row length vs size (is the config-5a slowdown the shape or the power cap?)
mkdir -p gpurun_out/r79
O=gpurun_out/r79
for i in 1 2; do for e in 2 0; do
  KS_LDG=$e python tools/time_paths.py 128 1024 16384 16 --reps 6 --paths fwd,dx >> $O/t.log 2>&1
  KS_LDG=$e python tools/time_paths.py 256 512 8192 16 --reps 6 --paths fwd,dx >> $O/t.log 2>&1
  KS_LDG=$e python tools/time_paths.py 512 1024 16384 16 --reps 4 --paths fwd,dx >> $O/t.log 2>&1
done; done
nvidia-smi --query-gpu=power.limit,power.draw,clocks.sm --format=csv >> $O/t.log
