# padded-TMA compute-bound kernels (stencil_pad, dw_pad): parity, A/B vs stencil_cb/dw_cb, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r22_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r22_pytest.log
for c in config4 config5b config2; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r22_pad_$c.json 2> gpurun_out/r22_pad_$c.err
done
KS_PAD_NS=2 KS_DWPAD_NS=2 timeout 600 python bench.py --config config4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r22_ns2_config4.json 2> gpurun_out/r22_ns2_config4.err
KS_PAD_NS=2 KS_DWPAD_NS=2 timeout 600 python bench.py --config config5b --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r22_ns2_config5b.json 2> gpurun_out/r22_ns2_config5b.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_pad|dw_pad" -s 2 -c 2 -o gpurun_out/r22_cb4 python tools/run_shape.py 256 256 2048 256 > gpurun_out/r22_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_pad|dw_pad" -s 2 -c 2 -o gpurun_out/r22_cb5b python tools/run_shape.py 32 1024 16384 128 > gpurun_out/r22_ncu2.log 2>&1
