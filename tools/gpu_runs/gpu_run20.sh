# ws stencil with balanced consumer warps (NT 128/256) and rows-per-tile: parity, sweep, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r20_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r20_pytest.log
KS_CB_NT=256 timeout 600 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x -k "warp_specialised or fwd_dx or full_config" > gpurun_out/r20_pytest256.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r20_pytest256.log
for c in config4 config5b; do
  for nt in 128 256; do
    KS_CB_NT=$nt timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r20_nt${nt}_$c.json 2> gpurun_out/r20_nt${nt}_$c.err
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_cb|dw_cb" -s 2 -c 2 -o gpurun_out/r20_cb4 python tools/run_shape.py 256 256 2048 256 > gpurun_out/r20_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_cb|dw_cb" -s 2 -c 2 -o gpurun_out/r20_cb5b python tools/run_shape.py 32 1024 16384 128 > gpurun_out/r20_ncu2.log 2>&1
