# dw_tma (16,8) single tap group for 8 < K <= 16 (config 5a)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r28_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r28_pytest.log
timeout 600 python bench.py --config config5a --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r28_j16_config5a.json 2>&1
KS_DWTMA_J16=0 timeout 600 python bench.py --config config5a --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r28_j8_config5a.json 2>&1
