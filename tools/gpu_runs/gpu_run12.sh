mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/ablation.py --out gpurun_out/ablation_paper > gpurun_out/ablation_paper.log 2>&1
timeout 600 python bench.py --config config1 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_config1.json 2> gpurun_out/bench_config1.err
