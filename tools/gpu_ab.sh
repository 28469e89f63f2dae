#!/bin/bash
# quick A/B of the long bench and the driver bench
TAG=${1:-ab}
OUT=gpurun_out
for i in 1 2; do
timeout 300 python bench.py --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e --no-replay > $OUT/b2000_${TAG}_$i.json 2>> $OUT/ab_$TAG.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/b20_${TAG}_$i.json 2>> $OUT/ab_$TAG.err
done
timeout 600 python -m pytest tests -m gpu -q --timeout 900 -rf -x -k "greed or paper_world or lab or tiny_free" > $OUT/ab_tests_$TAG.log 2>&1; echo tests=$? >> $OUT/ab_tests_$TAG.log
