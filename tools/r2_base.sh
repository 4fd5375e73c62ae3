set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_base_tests.log 2>&1; echo tests rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_base_bench.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/r2_base_tests.log
