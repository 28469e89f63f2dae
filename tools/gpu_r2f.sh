#!/bin/bash
# the paper world variants: bench (2000 steps and the driver's 20) and an ncu launch list of the co-located step
TAG=${1:-r2f}
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/status_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo build=$? >> $OUT/status_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo smoke=$? >> $OUT/status_$TAG.txt
for C in paper_world_coloc paper_world_cnn; do
  timeout 600 python bench.py --config $C --steps 2000 --warmup 5 > $OUT/bench_${C}_$TAG.json 2> $OUT/bench_${C}_$TAG.err; echo bench_$C=$? >> $OUT/status_$TAG.txt
done
CMD="python bench.py --config paper_world_coloc --steps 20 --warmup 300 --no-e2e --no-cpu-baseline --no-replay"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 200 --csv \
    --log-file $OUT/launches_coloc_$TAG.csv $CMD > $OUT/ncu_launch_coloc_$TAG.log 2>&1; echo ncu_launch=$? >> $OUT/status_$TAG.txt
cat $OUT/status_$TAG.txt
