mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "variants" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/ablation.py --out gpurun_out/ablation_paper > gpurun_out/ablation_paper.log 2>&1
timeout 900 python tools/ablation.py --shape 256 512 8192 7 --reps 5 --out gpurun_out/ablation_cfg3 > gpurun_out/ablation_cfg3.log 2>&1
