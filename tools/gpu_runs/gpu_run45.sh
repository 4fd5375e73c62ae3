mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r45_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r45_pytest.log
