#!/bin/bash
# Round-2 GPU job: smoke, GPU tests, the driver's bench (--steps 20 --warmup 5) and the long bench.
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/status_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo smoke=$? >> $OUT/status_$TAG.txt
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q --timeout 1200 -rf -s ${TESTS:-} > $OUT/gpu_tests_$TAG.log 2>&1; echo tests=$? >> $OUT/status_$TAG.txt
fi
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench20_$TAG.json 2> $OUT/bench20_$TAG.err; echo bench20=$? >> $OUT/status_$TAG.txt
if [ "${LONG:-1}" = "1" ]; then
  timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo bench=$? >> $OUT/status_$TAG.txt
fi
cat $OUT/status_$TAG.txt
