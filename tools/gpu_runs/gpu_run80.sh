# bwd_ldg (register-window fused backward): parity, A/B vs bwd_short at config 3 and K = 16, bench lines
mkdir -p gpurun_out/r80
O=gpurun_out/r80
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do for e in 1 0; do
  KS_BLDG=$e python tools/time_paths.py 256 512 8192 7 --reps 8 --paths bwd >> $O/t.log 2>&1
done; for e in 2 0; do
  KS_BLDG=$e python tools/time_paths.py 256 512 8192 16 --reps 8 --paths bwd >> $O/t.log 2>&1
done; done
for e in 0 1; do KS_BLDG=$e timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/c3_bldg$e.json 2>&1; done
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
