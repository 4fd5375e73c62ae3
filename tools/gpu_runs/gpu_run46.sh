mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -x -k "host or step" > gpurun_out/r46_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r46_pytest.log
for rep in 1 2; do
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/r46_bench_$rep.json 2> gpurun_out/r46_bench_$rep.err
done
