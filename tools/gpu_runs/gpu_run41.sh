# short rows: stencil_chan stage sweep vs stencil_rows; dw_rows 16x16 blocks vs 8x8
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r41_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r41_pytest.log
for ns in 1 2 3 4; do
  KS_CHAN_NS=$ns timeout 600 python tools/ablation.py --out gpurun_out/r41_chan_ns$ns > gpurun_out/r41_chan_ns$ns.log 2>&1
done
KS_ROWS_CHAN=0 KS_DWROWS_J8=1 timeout 600 python tools/ablation.py --out gpurun_out/r41_old > gpurun_out/r41_old.log 2>&1
