# Evidence refresh, part 1: final bench/tests/launch list + sanitizers (small outputs)
bash tools/gpu_final.sh
bash tools/gpu_sanitize.sh
