# stencil_ldg (register windows + 256-bit stores, full grid) for K <= 16: parity suite, A/B vs bwd_short stencils, bench lines
mkdir -p gpurun_out/r73
O=gpurun_out/r73
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do for e in 1 0; do
  KS_LDG=$e python tools/time_paths.py 256 512 8192 7 --reps 8 --paths fwd,dx >> $O/t.log 2>&1
  KS_LDG=$e python tools/time_paths.py 256 512 8192 16 --reps 8 --paths fwd,dx >> $O/t.log 2>&1
done; done
for c in config3 config5a; do
  for e in 0 1; do KS_LDG=$e timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/${c}_ldg$e.json 2>&1; done
done
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
