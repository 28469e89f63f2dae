#!/bin/bash
# A/B of library variants on one bench config: bash tools/gpu_abcfg.sh CONFIG STEPS v1 v2 ...
C=$1; K=$2; shift 2
OUT=gpurun_out
: > $OUT/abcfg.txt
for rep in 1 2; do for v in "$@"; do
  ECO_LIBSIM_OVERRIDE=build_var/libsim_$v.so timeout 600 python bench.py --config $C --steps $K --warmup 5 --no-cpu-baseline --no-e2e --no-replay > $OUT/abcfg_${v}_$rep.json 2>> $OUT/abcfg.err
  python -c "
import json; d=json.loads(open('$OUT/abcfg_${v}_$rep.json').read().strip().splitlines()[-1])
print('$v', '$C', $rep, round(d['ms_per_step']*1e3,2))" >> $OUT/abcfg.txt 2>&1
done; done
cat $OUT/abcfg.txt
