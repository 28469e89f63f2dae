#!/bin/bash
TAG=${1:-r2n}
OUT=gpurun_out
: > $OUT/status_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo smoke=$? >> $OUT/status_$TAG.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -rf -s > $OUT/gpu_tests_$TAG.log 2>&1; echo tests=$? >> $OUT/status_$TAG.txt
timeout 300 python bench.py --steps 20 --warmup 5 > $OUT/bench20_$TAG.json 2> $OUT/bench20_$TAG.err; echo bench20=$? >> $OUT/status_$TAG.txt
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo bench=$? >> $OUT/status_$TAG.txt
cat $OUT/status_$TAG.txt
