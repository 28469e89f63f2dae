#!/bin/bash
# A/B of library variants on the large world at its cap and the ensemble
OUT=gpurun_out
: > $OUT/ablarge.txt
for v in "$@"; do
  ECO_LIBSIM_OVERRIDE=build_var/libsim_$v.so timeout 600 python bench.py --config large_world --steps 10 --warmup 300 --no-cpu-baseline --no-e2e --no-replay > $OUT/ablarge_$v.json 2>> $OUT/ablarge.err
  ECO_LIBSIM_OVERRIDE=build_var/libsim_$v.so timeout 600 python bench.py --config ensemble --steps 20 --warmup 20 --no-cpu-baseline --no-e2e --no-replay > $OUT/abens_$v.json 2>> $OUT/ablarge.err
  python -c "
import json
a=json.loads(open('$OUT/ablarge_$v.json').read().strip().splitlines()[-1]); b=json.loads(open('$OUT/abens_$v.json').read().strip().splitlines()[-1])
print('$v', 'large', round(a['ms_per_step'],4), 'ensemble', round(b['ms_per_step'],4))" >> $OUT/ablarge.txt 2>&1
done
cat $OUT/ablarge.txt
