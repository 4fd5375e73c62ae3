#!/bin/bash
# Copy the final evidence run (tools/gpu_final.sh -> gpurun_out/final) into profiles/.
set -e
O=gpurun_out/final
for c in config1 config2 config3 config4 config5a config5b config5c config3_pairwise; do
  [ -s $O/bench_$c.json ] && tail -n1 $O/bench_$c.json > profiles/r01_bench_$c.json
done
[ -s $O/bench_reference.json ] && tail -n1 $O/bench_reference.json > profiles/r01_bench_reference_config3.json
for a in paper_shape config3; do
  [ -s $O/ablation_$a.md ] && cp $O/ablation_$a.md profiles/r01_ablation_$a.md && cp $O/ablation_$a.csv profiles/r01_ablation_$a.csv
done
[ -s $O/launches.csv ] && python tools/ncu_summary.py r01 --launches $O/launches.csv
echo collected
