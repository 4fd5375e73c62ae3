# stencil_pad producer-lane vs CTA-barrier refill, per config
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x -k "fwd_dx or padded or full_config" > gpurun_out/r24_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r24_pytest.log
KS_PAD_PROD=0 timeout 600 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x -k "fwd_dx or padded" > gpurun_out/r24_pytest_bar.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r24_pytest_bar.log
for c in config2 config4 config5b; do
  for pr in 0 1; do
    KS_PAD_PROD=$pr timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r24_p${pr}_$c.json 2> gpurun_out/r24_p${pr}_$c.err
  done
done
