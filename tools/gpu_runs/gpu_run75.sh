# Evidence refresh after stencil_ldg: final bench/tests/launch list + sanitizers + ncu capture of the config-3 stencils
bash tools/gpu_final.sh
bash tools/gpu_sanitize.sh
O=gpurun_out/ncu75
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stencil_ldg|bwd_short" -c 4 -o /tmp/ldg3 python tools/run_shape.py 256 512 8192 7 --reps 1 --bwd > $O/ldg3.log 2>&1
ncu -i /tmp/ldg3.ncu-rep --page raw --csv > $O/ldg3.csv 2>> $O/ldg3.log
ncu -i /tmp/ldg3.ncu-rep --page details --csv > $O/ldg3_details.csv 2>> $O/ldg3.log
