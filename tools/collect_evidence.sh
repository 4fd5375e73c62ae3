#!/bin/bash
# Copy the evidence run (tools/gpu_evidence.sh -> gpurun_out/ev) into profiles/ (committed).
set -e
O=gpurun_out/ev; P=profiles
for f in $O/bench_*.json; do
  b=$(basename $f .json)
  [ -s $f ] && tail -n1 $f > $P/r02_$b.json || true
done
[ -s $O/plans.json ] && cp $O/plans.json $P/r02_plans.json
[ -s $O/b200_device_spec.json ] && cp $O/b200_device_spec.json $P/b200_device_spec.json
for a in paper_shape config3; do
  for s in .md _paper.csv _library.csv; do [ -s $O/ablation_$a$s ] && cp $O/ablation_$a$s $P/r02_ablation_$a$s; done
done
for c in "config2 64 128 4096 4096" "config3 256 512 8192 7" "config4 1024 256 2048 256" "config5a 512 1024 16384 16" "config5b 512 1024 16384 128" "config5c_g8 64 1024 16384 1024"; do
  set -- $c
  [ -s $O/launches_$1.csv ] && python tools/ncu_summary.py r02 --config $1 --shape $2 $3 $4 $5 --run-shape $O/launches_$1.csv
done
[ -s $O/launches_bench.csv ] && python tools/ncu_summary.py r02 --launches $O/launches_bench.csv --config bench_config3 || true
for r in config3 config2 config4 config5a; do
  [ -s $O/full_$r.raw.csv ] && python tools/ncu_summary.py r02 --full $r=$O/full_$r.raw.csv
done
for t in memcheck racecheck synccheck; do [ -s $O/sanitize_$t.log ] && tail -n 3 $O/sanitize_$t.log > $P/r02_sanitize_$t.log; done
[ -s $O/pytest_gpu.log ] && tail -n 2 $O/pytest_gpu.log > $P/r02_pytest_gpu.log
[ -s $O/smoke.log ] && cp $O/smoke.log $P/r02_smoke.log
[ -s $O/hbm_mix.log ] && (echo "# tools/probes/hbm_mix_probe.cu (tools/gpu_evidence.sh): HBM streaming rate per read:write mix"; cat $O/hbm_mix.log) > $P/r02_hbm_mix.txt
# the reference's own analysis pipeline over the ablation logs (oracle/_ref/ks_b200_report)
if [ -x oracle/_ref/ks_b200_report ]; then
  for l in $P/r02_ablation_*_paper.csv $P/r02_ablation_*_library.csv; do
    [ -s $l ] || continue
    n=$(basename $l .csv); d=$P/r02_refreport_${n#r02_ablation_}; mkdir -p $d
    shape=$(head -1 $l | sed 's/.*(B,H,L,K)=(\([0-9,]*\)).*/\1/' | tr ',' ' ')
    oracle/_ref/ks_b200_report $l $P/b200_device_spec.json $shape $d > /dev/null
  done
fi
echo collected
