#!/bin/bash
# Regrowth tests, the configs[2] microbenchmark and ncu captures of k_regrow_tiled.
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/status_regrow_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 1200 -rf -s -k "regrowth or large_world_full_size or large_grid" > $OUT/gpu_tests_regrow_$TAG.log 2>&1; echo tests=$? >> $OUT/status_regrow_$TAG.txt
timeout 900 python tools/bench_regrowth.py --out $OUT/regrowth_$TAG.json > /dev/null 2> $OUT/regrowth_$TAG.err; echo regrowth=$? >> $OUT/status_regrow_$TAG.txt
timeout 300 python tools/profile_regrow.py --steps 25 > $OUT/prof_regrow_plain_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_regrow_tiled -s 20 -c 1 -o $OUT/prof_regrow_growth_$TAG python tools/profile_regrow.py --steps 25 > $OUT/ncu_regrow_growth_$TAG.log 2>&1; echo ncu_growth=$? >> $OUT/status_regrow_$TAG.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_regrow_tiled -s 900 -c 1 -o $OUT/prof_regrow_sat_$TAG python tools/profile_regrow.py --steps 905 > $OUT/ncu_regrow_sat_$TAG.log 2>&1; echo ncu_sat=$? >> $OUT/status_regrow_$TAG.txt
cat $OUT/status_regrow_$TAG.txt
