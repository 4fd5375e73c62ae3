O=gpurun_out/p3; mkdir -p $O
python tools/dump_plans.py $O/plans.json > $O/plans.log 2>&1
python tools/time_paths.py 256 512 8192 7 --mode separate --reps 20 --paths fwd,dx,dw,bwd > $O/time_c3.log 2>&1
python tools/time_paths.py 512 1024 16384 16 --mode separate --reps 5 > $O/time_c5a.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
tail -2 $O/gpu_tests.log
