# un-narrowable 128-bit shared loads (lds4): parity + configs 3 / 5a / paper shape timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r38_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r38_pytest.log
for c in config3 config5a config4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r38_$c.json 2>&1
done
timeout 900 python tools/ablation.py --out gpurun_out/r38_ablation > gpurun_out/r38_ablation.log 2>&1
