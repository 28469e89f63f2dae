#!/bin/bash
# A/B of library variants over several bench configs, interleaved, REPS repetitions:
#   bash tools/gpu_ab_multi.sh REPS "cfg:steps cfg:steps ..." v1 v2 ...
REPS=$1; CFGS=$2; shift 2
OUT=gpurun_out
: > $OUT/abm.txt
for rep in $(seq 1 $REPS); do for cs in $CFGS; do for v in "$@"; do
  C=${cs%%:*}; K=${cs##*:}
  ECO_LIBSIM_OVERRIDE=build_var/libsim_$v.so timeout 600 python bench.py --config $C --steps $K --warmup 5 --no-cpu-baseline --no-e2e --no-replay > $OUT/abm_${v}_${C}_$rep.json 2>> $OUT/abm.err
  python -c "
import json; d=json.loads(open('$OUT/abm_${v}_${C}_$rep.json').read().strip().splitlines()[-1])
print('$v', '$C', $K, $rep, round(d['ms_per_step']*1e3,2))" >> $OUT/abm.txt 2>&1
done; done; done
cat $OUT/abm.txt
