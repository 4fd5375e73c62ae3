# dw_tma producer-lane (no CTA barrier per item) vs barrier; stencil_tma NS=4 at 5a
mkdir -p gpurun_out
KS_DWTMA_PROD=1 timeout 600 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x -k "hierarchical or full_config" > gpurun_out/r27_pytest_prod.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r27_pytest_prod.log
for c in config3 config5a; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r27_base_$c.json 2>&1
  KS_DWTMA_PROD=1 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r27_prod_$c.json 2>&1
  KS_STENCIL_NS=4 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r27_ns4_$c.json 2>&1
done
