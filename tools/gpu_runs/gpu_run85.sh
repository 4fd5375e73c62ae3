# stencil_ldgk (long-K register windows, uniform taps) vs stencil_pad: parity + timing on the compute-bound configs
mkdir -p gpurun_out/r85
O=gpurun_out/r85
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -k "ldgk" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do for e in 1 0; do
  KS_LDGK=$e python tools/time_paths.py 1024 256 2048 256 --reps 6 --paths fwd,dx >> $O/t.log 2>&1
  KS_LDGK=$e python tools/time_paths.py 128 1024 16384 128 --reps 4 --paths fwd,dx >> $O/t.log 2>&1
  KS_LDGK=$e python tools/time_paths.py 64 128 4096 4096 --reps 6 --paths fwd,dx >> $O/t.log 2>&1
  KS_LDGK=$e python tools/time_paths.py 64 1024 16384 1024 --reps 3 --paths fwd,dx >> $O/t.log 2>&1
  KS_LDGK=$e python tools/time_paths.py 16 64 1024 64 --reps 20 --paths fwd,dx >> $O/t.log 2>&1
done; done
