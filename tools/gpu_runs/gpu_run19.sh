# warp-specialised compute-bound kernels: parity, then A/B vs the single-role kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r19_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r19_pytest.log
for c in config4 config5b config2; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r19_ws_$c.json 2> gpurun_out/r19_ws_$c.err
  KS_STENCIL_WS=0 KS_DW_WS=0 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r19_old_$c.json 2> gpurun_out/r19_old_$c.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_cb|dw_cb" -s 2 -c 2 -o gpurun_out/r19_cb4 python tools/run_shape.py 256 256 2048 256 > gpurun_out/r19_ncu.log 2>&1
