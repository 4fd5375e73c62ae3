#!/bin/bash
# Refresh the committed evidence on ONE GPU (never multi-rank under ncu):
#   gpurun --timeout 3600 -- 'bash tools/gpu_evidence.sh'   then   bash tools/collect_evidence.sh
O=gpurun_out/ev; mkdir -p $O
T="timeout 900"
$T python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
python tools/dump_plans.py $O/plans.json > $O/plans.log 2>&1
# the suite below checks the library against the plans it just dumped (collect_evidence.sh commits them)
[ -s $O/plans.json ] && cp $O/plans.json profiles/r02_plans.json
python tools/b200_device_spec.py $O/b200_device_spec.json > $O/spec.log 2>&1
# HBM streaming rate per read:write mix (the roof each HBM-bound path is judged against)
[ -x tools/probes/hbm_mix_probe ] && timeout 120 tools/probes/hbm_mix_probe > $O/hbm_mix.log 2>&1
# bench lines: the headline (config 3, Separate = the reference's default, e2e + CPU baseline), then every config in both modes
$T python bench.py > $O/bench_config3.json 2> $O/bench_config3.err
$T python bench.py --impl reference > $O/bench_reference_config3.json 2> $O/bench_reference_config3.err
for m in separate fused; do
  for c in config1 config2 config3 config4 config5a config5b; do
    $T python bench.py --config $c --mode $m --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_${c}_$m.json 2> $O/bench_${c}_$m.err
  done
  $T python bench.py --config config5c --mode $m --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_config5c_$m.json 2> $O/bench_config5c_$m.err
done
$T python bench.py --scheme pairwise --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_config3_pairwise.json 2> $O/bench_config3_pairwise.err
$T python bench.py --config config4 --global-batch 1024 --mode fused --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_config4_strong_n1.json 2> $O/bench_config4_strong_n1.err
# the N > 1 code path on this one GPU: 2 ranks, gloo + the library's host communicator
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633"
$T $TR bench.py --gpus 2 --steps 5 --warmup 3 --transport host --no-e2e --no-cpu-baseline > $O/bench_n2host_config3.json 2> $O/bench_n2host_config3.err
$T $TR bench.py --gpus 2 --steps 5 --warmup 3 --transport host --combine peer --config config4 --global-batch 1024 --mode fused --no-e2e --no-cpu-baseline > $O/bench_n2host_config4_peer.json 2> $O/bench_n2host_config4_peer.err
# the paper's ablation on B200 (timing logs in the reference's CSV schema)
$T python tools/ablation.py --out $O/ablation_paper_shape > $O/ablation_paper.log 2>&1
$T python tools/ablation.py --shape 256 512 8192 7 --reps 5 --out $O/ablation_config3 > $O/ablation_config3.log 2>&1
# ncu: per-config launch lists (DRAM bytes, geometry) and full captures of the dominant kernels
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size,launch__shared_mem_per_block_dynamic
for c in "config2 64 128 4096 4096" "config3 256 512 8192 7" "config4 1024 256 2048 256" "config5a 512 1024 16384 16" "config5b 512 1024 16384 128" "config5c_g8 64 1024 16384 1024"; do
  set -- $c
  $T ncu --metrics $M --clock-control none --csv --log-file $O/launches_$1.csv python tools/run_shape.py $2 $3 $4 $5 --reps 1 --bwd > $O/ncu_launch_$1.log 2>&1
done
$T ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_bench.log 2>&1
$T ncu --set full --clock-control none --import-source on -k regex:"bwd_short|stencil_ldg" -s 4 -c 4 -o $O/full_config3 python tools/run_shape.py 256 512 8192 7 --reps 2 --bwd > $O/ncu_full3.log 2>&1
$T ncu --set full --clock-control none --import-source on -k regex:"stencil_pad|dw_pad" -s 3 -c 3 -o $O/full_config2 python tools/run_shape.py 16 128 4096 4096 --reps 2 --mode fused > $O/ncu_full2.log 2>&1
$T ncu --set full --clock-control none --import-source on -k regex:"stencil_pad|dw_pad" -s 3 -c 3 -o $O/full_config4 python tools/run_shape.py 256 256 2048 256 --reps 2 --mode fused > $O/ncu_full4.log 2>&1
$T ncu --set full --clock-control none --import-source on -k regex:"bwd_short" -s 4 -c 4 -o $O/full_config5a python tools/run_shape.py 64 1024 16384 16 --reps 2 --bwd > $O/ncu_full5a.log 2>&1
for r in full_config3 full_config2 full_config4 full_config5a; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/$r.raw.csv 2>/dev/null
  rm -f $O/$r.ncu-rep  # gpurun copies back at most 64 MiB
done
# sanitizers on the small cases (TMA rings, mbarriers, the mirrored stencil, unaligned staging)
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/sanitize_$tool.log
done
$T python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
ls -la $O
