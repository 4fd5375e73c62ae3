# Round-2 GPU check: the new multi-rank / alignment / config-5 tests first, then the whole -m gpu suite,
# then short bench lines in both multiply-add modes.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multirank_gpu.py -x -q > gpurun_out/r2_multirank.log 2>&1; echo multirank rc=$?
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "unaligned or config5" > gpurun_out/r2_align_cfg5.log 2>&1; echo align rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_gpu_all.log 2>&1; echo all rc=$?
for m in separate fused; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --mode $m > gpurun_out/r2_bench_$m.log 2>&1; echo bench $m rc=$?
done
tail -3 gpurun_out/r2_multirank.log gpurun_out/r2_align_cfg5.log gpurun_out/r2_gpu_all.log
