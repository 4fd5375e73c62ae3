# direct 256-bit stores for the short-kernel stencil / fused-backward outputs: parity, A/B vs TMA store
mkdir -p gpurun_out/r58
O=gpurun_out/r58
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for K in 7 16; do
  KS_DST=0 python tools/time_paths.py 256 512 8192 $K --reps 10 >> $O/t.log 2>&1
  python tools/time_paths.py 256 512 8192 $K --reps 10 >> $O/t.log 2>&1
done
