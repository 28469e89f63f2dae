#!/bin/bash
TAG=${1:-r2k}
OUT=gpurun_out
: > $OUT/status_$TAG.txt
timeout 900 python -m pytest tests/test_gpu_banded.py tests/test_gpu_checks.py -q --timeout 900 -rf -s -x > $OUT/tests_$TAG.log 2>&1; echo tests=$? >> $OUT/status_$TAG.txt
timeout 1200 python tools/band_scaling.py --out $OUT/band_scaling_$TAG.json > /dev/null 2> $OUT/band_scaling_$TAG.err; echo band_scaling=$? >> $OUT/status_$TAG.txt
SKIP=$((160*8*18)) COUNT=150 bash tools/gpu_band_prof.sh $TAG; echo prof=$? >> $OUT/status_$TAG.txt
cat $OUT/status_$TAG.txt
