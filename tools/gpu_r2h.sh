#!/bin/bash
TAG=${1:-r2h}
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/status_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo smoke=$? >> $OUT/status_$TAG.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 900 -rf -s -k "regrowth or banded or tiny or init" > $OUT/tests_$TAG.log 2>&1; echo tests=$? >> $OUT/status_$TAG.txt
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench20_persist_${TAG}_$i.json 2> $OUT/bench20_persist_$TAG.err; echo bench20_persist=$? >> $OUT/status_$TAG.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-l2-persist > $OUT/bench20_nopersist_${TAG}_$i.json 2> $OUT/bench20_nopersist_$TAG.err; echo bench20_nopersist=$? >> $OUT/status_$TAG.txt
done
timeout 600 python bench.py --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench2000_persist_$TAG.json 2> $OUT/bench2000_$TAG.err; echo bench2000=$? >> $OUT/status_$TAG.txt
timeout 600 python bench.py --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e --no-l2-persist > $OUT/bench2000_nopersist_$TAG.json 2>> $OUT/bench2000_$TAG.err; echo bench2000n=$? >> $OUT/status_$TAG.txt
timeout 600 python tools/bench_regrowth.py --out $OUT/regrowth_$TAG.json > /dev/null 2> $OUT/regrowth_$TAG.err; echo regrowth=$? >> $OUT/status_$TAG.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_regrow_tiled -s 20 -c 1 -o $OUT/prof_regrow_growth_$TAG python tools/profile_regrow.py --steps 25 > $OUT/ncu_g_$TAG.log 2>&1; echo ncu_growth=$? >> $OUT/status_$TAG.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_regrow_tiled -s 900 -c 1 -o $OUT/prof_regrow_sat_$TAG python tools/profile_regrow.py --steps 905 > $OUT/ncu_s_$TAG.log 2>&1; echo ncu_sat=$? >> $OUT/status_$TAG.txt
timeout 1200 python tools/band_scaling.py --out $OUT/band_scaling_$TAG.json > /dev/null 2> $OUT/band_scaling_$TAG.err; echo band_scaling=$? >> $OUT/status_$TAG.txt
cat $OUT/status_$TAG.txt
