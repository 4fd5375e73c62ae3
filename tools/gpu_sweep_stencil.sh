mkdir -p gpurun_out
for nt in 256 128; do for ns in 2 3 4 6 8; do
  echo "NT=$nt NS=$ns" >> gpurun_out/sweep.txt
  KS_STENCIL_NT=$nt KS_STENCIL_NS=$ns timeout 300 python bench.py --config config3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['paths']['fwd'], d['paths']['dX'])" >> gpurun_out/sweep.txt
done; done
