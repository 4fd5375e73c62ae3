# ABAB: zero-halo skipping on/off at configs 4 and 5b (does the skip logic cost anything where it never fires?)
mkdir -p gpurun_out/r67
O=gpurun_out/r67
for i in 1 2; do for s in 1 0; do
  KS_PAD_SKIP=$s python tools/time_paths.py 1024 256 2048 256 --reps 8 --paths fwd,dx,dw >> $O/t.log 2>&1
  KS_PAD_SKIP=$s python tools/time_paths.py 128 1024 16384 128 --reps 5 --paths fwd,dx,dw >> $O/t.log 2>&1
done; done
