mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "pairwise or full_config or step_host" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config config3 --scheme pairwise --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_config3_pw.json 2> gpurun_out/bench_config3_pw.err
timeout 600 python bench.py --config config2 --scheme pairwise --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_config2_pw.json 2> gpurun_out/bench_config2_pw.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_tma -s 1 -c 1 -o gpurun_out/prof_stencil_c4 python bench.py --config config4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dw_pairwise -s 1 -c 1 -o gpurun_out/prof_pw_c3 python bench.py --config config3 --scheme pairwise --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pw.log 2>&1
