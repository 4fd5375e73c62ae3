# Full evidence refresh: GPU suite, smoke, every bench line, pairwise + reference arms, ablations, launch list
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_config3.json 2> $O/bench_config3.err
for c in config1 config2 config4 config5a config5b; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --config config5c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_config5c.json 2> $O/bench_config5c.err
timeout 600 python bench.py --scheme pairwise --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_config3_pairwise.json 2> $O/bench_config3_pairwise.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python tools/ablation.py --out $O/ablation_paper_shape > $O/ablation_paper.log 2>&1
timeout 900 python tools/ablation.py --shape 256 512 8192 7 --reps 5 --out $O/ablation_config3 > $O/ablation_config3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 250 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/launches.log 2>&1
