#!/bin/bash
# A/B of an environment switch on bench configs: bash tools/gpu_ab_env.sh VAR "v1 v2" "cfg:steps:warmup ..."
VAR=$1; VALS=$2; CFGS=$3
OUT=gpurun_out
: > $OUT/abe.txt
for rep in 1 2; do for cs in $CFGS; do for v in $VALS; do
  IFS=: read C K W <<< "$cs"
  env $VAR=$v timeout 900 python bench.py --config $C --steps $K --warmup $W --no-cpu-baseline --no-e2e --no-replay > $OUT/abe_${v}_${C}_${W}_$rep.json 2>> $OUT/abe.err
  python -c "
import json; d=json.loads(open('$OUT/abe_${v}_${C}_${W}_$rep.json').read().strip().splitlines()[-1])
print('$VAR=$v', '$C', 't=$W+$K', $rep, round(d['ms_per_step']*1e3,2), 'agents', d.get('agents_mean'))" >> $OUT/abe.txt 2>&1
done; done; done
cat $OUT/abe.txt
