# FFMA2 (packed pair FMA) in stencil_pad's Fused inner loop: parity + compute-bound configs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r48_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r48_pytest.log
for c in config2 config4 config5b; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r48_$c.json 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stencil_pad" -s 1 -c 1 -o gpurun_out/r48_pad4 python tools/run_shape.py 256 256 2048 256 > gpurun_out/r48_ncu.log 2>&1
