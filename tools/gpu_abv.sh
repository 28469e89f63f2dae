#!/bin/bash
# A/B of library variants in build_var/ (ECO_LIBSIM_OVERRIDE): the bench at the driver's
# settings (t = 5..25) twice and over 2000 steps, per variant, interleaved.
# Usage: bash tools/gpu_abv.sh TAG v1 v2 ...
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/abv_$TAG.txt
for rep in 1 2; do
for v in "$@"; do
  L=build_var/libsim_$v.so
  ECO_LIBSIM_OVERRIDE=$L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/abv_${TAG}_${v}_20_$rep.json 2>> $OUT/abv_$TAG.err
  ECO_LIBSIM_OVERRIDE=$L timeout 300 python bench.py --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e --no-replay > $OUT/abv_${TAG}_${v}_2000_$rep.json 2>> $OUT/abv_$TAG.err
  for n in 20 2000; do python -c "
import json; d=json.loads(open('$OUT/abv_${TAG}_${v}_${n}_$rep.json').read().strip().splitlines()[-1])
print('$v', $n, $rep, round(d['ms_per_step']*1e3,2), d.get('graph_kernel_ms_per_step'), d.get('post_phase_us_per_step'))" >> $OUT/abv_$TAG.txt 2>&1; done
done
done
cat $OUT/abv_$TAG.txt
