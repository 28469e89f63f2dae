#!/bin/bash
TAG=${1:-r2g2}
OUT=gpurun_out
: > $OUT/status_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo build=$? >> $OUT/status_$TAG.txt
timeout 900 python -m pytest tests/test_gpu_coloc.py tests/test_gpu_checks.py -x -q -rf -s --timeout 600 > $OUT/co_$TAG.log 2>&1; echo co=$? >> $OUT/status_$TAG.txt
timeout 600 python bench.py --config paper_world_coloc --steps 2000 --warmup 5 > $OUT/bench_coloc_$TAG.json 2> $OUT/bench_coloc_$TAG.err; echo bench=$? >> $OUT/status_$TAG.txt
# one banded G=8 step's kernels (every band): 160 warm-up steps, then the launch list of one step
SKIP=0 COUNT=100000 G=8 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 6000 --csv --log-file $OUT/band_launches_$TAG.csv python tools/profile_band.py --G 8 --warmup 20 --steps 1 > $OUT/band_prof_$TAG.log 2>&1; echo band_prof=$? >> $OUT/status_$TAG.txt
cat $OUT/status_$TAG.txt
