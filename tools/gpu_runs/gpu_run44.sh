# stencil_tma 128-thread / 2-stage tiles for K > 8: parity + config 5a / 3 lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r44_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r44_pytest.log
timeout 600 python bench.py --config config5a --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r44_config5a.json 2>&1
timeout 600 python bench.py --config config3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r44_config3.json 2>&1
KS_STENCIL_NT=128 KS_STENCIL_NS=2 timeout 600 python bench.py --config config3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r44_config3_nt128ns2.json 2>&1
