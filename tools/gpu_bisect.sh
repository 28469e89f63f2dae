#!/bin/bash
# 10,000-step bench of earlier commits' builds (bisect/<sha>/, each with its own bench.py)
OUT=$PWD/gpurun_out
: > $OUT/bisect.txt
for rep in 1 2; do
for c in "$@"; do
  (cd bisect/$c && timeout 300 python bench.py --steps 10000 --warmup 5 --no-cpu-baseline --no-e2e --no-replay > $OUT/bisect_${c}_$rep.json 2>> $OUT/bisect.err)
  python -c "
import json; d=json.loads(open('$OUT/bisect_${c}_$rep.json').read().strip().splitlines()[-1])
print('$c', $rep, round(d['ms_per_step']*1e3,2), d.get('post_phase_us_per_step'))" >> $OUT/bisect.txt 2>&1
done; done
cat $OUT/bisect.txt
