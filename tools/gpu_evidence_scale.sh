#!/bin/bash
# ncu --set full of one step of the large world at its cap and of the 64-world ensemble
TAG=${1:-r2z}
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/status_scale_$TAG.txt
for C in large_world:300 ensemble:20; do
  N=${C%%:*}; W=${C##*:}
  PCMD="python tools/profile_step.py --config $N --warmup $W --out $OUT/step_${N}_$TAG.json"
  timeout 600 $PCMD > $OUT/plain_${N}_$TAG.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_policy_half|k_prepare_p|k_post" -s $((2 * W)) -c 3 \
      -o $OUT/prof_${N}_$TAG $PCMD > $OUT/ncu_${N}_$TAG.log 2>&1 && \
  python tools/ncu_summary.py $OUT/prof_${N}_$TAG.ncu-rep --step $OUT/step_${N}_$TAG.json --out $OUT/ncu_summary_${N}_$TAG.json > /dev/null 2>&1
  echo ncu_$N=$? >> $OUT/status_scale_$TAG.txt
done
cat $OUT/status_scale_$TAG.txt
