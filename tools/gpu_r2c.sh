#!/bin/bash
# network 1 (the paper's CNN-LSTM): smoke, bench of paper_world_cnn and paper_world, ncu of one step
TAG=${1:-r2c}
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/status_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo build=$? >> $OUT/status_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo smoke=$? >> $OUT/status_$TAG.txt
for C in paper_world_cnn paper_world; do
  timeout 600 python bench.py --config $C --steps 2000 --warmup 5 > $OUT/bench_${C}_$TAG.json 2> $OUT/bench_${C}_$TAG.err; echo bench_$C=$? >> $OUT/status_$TAG.txt
done
W=300
PCMD="python tools/profile_step.py --config paper_world_cnn --warmup $W --out $OUT/step_cnn_$TAG.json"
timeout 300 $PCMD > $OUT/plain_cnn_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_policy_cnn|k_post" -s $((2 * W - 1)) -c 2 \
    -o $OUT/prof_cnn_$TAG $PCMD > $OUT/ncu_cnn_$TAG.log 2>&1 && \
python tools/ncu_summary.py $OUT/prof_cnn_$TAG.ncu-rep --step $OUT/step_cnn_$TAG.json --out $OUT/ncu_summary_cnn_$TAG.json > /dev/null 2>&1
echo ncu_cnn=$? >> $OUT/status_$TAG.txt
cat $OUT/status_$TAG.txt
