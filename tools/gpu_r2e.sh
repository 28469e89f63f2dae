#!/bin/bash
# round-2 evidence: banded-world scaling estimate, regrowth ncu captures (growth / saturated),
# agent-sharded scaling estimate, checked build (incl. the CNN world), banded launch list
TAG=${1:-r2e}
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/status_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo build=$? >> $OUT/status_$TAG.txt
timeout 900 python -m pytest tests/test_gpu_checks.py -q --timeout 900 -rf > $OUT/checks_$TAG.log 2>&1; echo checks=$? >> $OUT/status_$TAG.txt
timeout 1500 python tools/band_scaling.py --out $OUT/band_scaling_$TAG.json > /dev/null 2> $OUT/band_scaling_$TAG.err; echo band_scaling=$? >> $OUT/status_$TAG.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_regrow_tiled -s 20 -c 1 -o $OUT/prof_regrow_growth_$TAG python tools/profile_regrow.py --steps 25 > $OUT/ncu_g_$TAG.log 2>&1; echo ncu_growth=$? >> $OUT/status_$TAG.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_regrow_tiled -s 900 -c 1 -o $OUT/prof_regrow_sat_$TAG python tools/profile_regrow.py --steps 905 > $OUT/ncu_s_$TAG.log 2>&1; echo ncu_sat=$? >> $OUT/status_$TAG.txt
timeout 900 python tools/shard_scaling.py --ranks 1,2,4,8 > $OUT/shard_scaling_$TAG.json 2> $OUT/shard_scaling_$TAG.err; echo shard_scaling=$? >> $OUT/status_$TAG.txt
cat $OUT/status_$TAG.txt
