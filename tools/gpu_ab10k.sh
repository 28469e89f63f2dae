#!/bin/bash
OUT=gpurun_out
: > $OUT/ab10k.txt
for rep in 1 2; do
for v in "$@"; do
  ECO_LIBSIM_OVERRIDE=build_var/libsim_$v.so timeout 300 python bench.py --steps 10000 --warmup 5 --no-cpu-baseline --no-e2e --no-replay > $OUT/ab10k_${v}_$rep.json 2>> $OUT/ab10k.err
  python -c "
import json; d=json.loads(open('$OUT/ab10k_${v}_$rep.json').read().strip().splitlines()[-1])
print('$v', $rep, round(d['ms_per_step']*1e3,2), d.get('post_phase_us_per_step'))" >> $OUT/ab10k.txt 2>&1
done; done
cat $OUT/ab10k.txt
