# plans (carveout), config-1 fwd dispatch debug, stage-count A/B of the short-K dW / fused backward, ncu DRAM
# launch lists at the full configs
O=gpurun_out/p2; mkdir -p $O
python tools/dump_plans.py $O/plans.json > $O/plans.log 2>&1
python - > $O/c1debug.log 2>&1 <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2604_25422_b200 as ks
for shp in [(16,64,1024,64),(16,64,2048,64),(16,32,1024,64),(8,64,1024,64),(16,64,1024,63),(16,64,1024,65)]:
    for p in ('fwd','dx'):
        print(shp,p,[(r['kernel'][:40],r['grid'][0],r['block'][0],r['smem']) for r in ks.plan(p,*shp)])
with ks.options(stencil_pad=0):
    print('stencil_pad=0', [(r['kernel'][:40],r['grid'][0],r['smem']) for r in ks.plan('fwd',16,64,1024,64)])
PY
for v in default fns3 fns5 dwns6; do
  for m in separate fused; do
    if [ $v = default ]; then L=""; else L=build/variants/$v/libks_dwconv1d.so; fi
    echo "== $v $m" >> $O/ab.log
    KS_LIB=$L python tools/time_paths.py 256 512 8192 7 --mode $m --reps 20 --paths dw,bwd >> $O/ab.log 2>&1
  done
done
for c in "64 128 4096 4096" "1024 256 2048 256" "512 1024 16384 16" "512 1024 16384 128" "256 512 8192 7"; do
  n=$(echo $c | tr ' ' _)
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size,launch__shared_mem_per_block_dynamic --clock-control none --csv --log-file $O/launches_$n.csv python tools/run_shape.py $c --reps 1 --bwd > $O/ncu_$n.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size,launch__shared_mem_per_block_dynamic --clock-control none --csv --log-file $O/launches_512_1024_16384_1024.csv python tools/run_shape.py 64 1024 16384 1024 --reps 1 --bwd > $O/ncu_5c.log 2>&1
ls -la $O
