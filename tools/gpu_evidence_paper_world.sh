#!/bin/bash
# ncu --set full of one step of the paper's world with the paper's network, exclusive and
# co-located (k_policy_cnn_blk, k_post / k_co_move, k_co_live, k_co_rank)
TAG=${1:-r2g}
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/status_$TAG.txt
W=300
for C in paper_world_cnn paper_world_coloc; do
  PCMD="python tools/profile_step.py --config $C --warmup $W --out $OUT/step_${C}_$TAG.json"
  timeout 300 $PCMD > $OUT/plain_${C}_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_policy_cnn|k_post|k_co_" -s $((2 * W - 1)) -c 4 \
      -o $OUT/prof_${C}_$TAG $PCMD > $OUT/ncu_${C}_$TAG.log 2>&1 && \
  python tools/ncu_summary.py $OUT/prof_${C}_$TAG.ncu-rep --step $OUT/step_${C}_$TAG.json --out $OUT/ncu_summary_${C}_$TAG.json > /dev/null 2>&1
  echo ncu_$C=$? >> $OUT/status_$TAG.txt
done
cat $OUT/status_$TAG.txt
