# channel-major short-row stencil: parity + paper-shape ablation
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r40_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r40_pytest.log
timeout 900 python tools/ablation.py --out gpurun_out/r40_ablation > gpurun_out/r40_ablation.log 2>&1
KS_ROWS_CHAN=0 timeout 900 python tools/ablation.py --out gpurun_out/r40_ablation_old > gpurun_out/r40_ablation_old.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stencil_chan|dw_rows" -s 2 -c 2 -o gpurun_out/r40_chan python tools/run_shape.py 16384 128 48 48 > gpurun_out/r40_ncu.log 2>&1
