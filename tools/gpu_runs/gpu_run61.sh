# ABAB: TMA-store vs direct-store stencils inside the config-5a bench (power-capped, long run)
mkdir -p gpurun_out/r61
O=gpurun_out/r61
for i in 1 2; do
  for d in 0 1; do
    KS_DST=$d timeout 600 python bench.py --config config5a --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/5a_dst${d}_$i.json 2>&1
  done
done
for d in 0 1; do KS_DST=$d python tools/time_paths.py 512 1024 16384 16 --reps 5 --paths fwd,dx >> $O/t.log 2>&1; done
