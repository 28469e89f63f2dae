#!/bin/bash
# Measurement job: smoke, the whole -m gpu suite, the bench at the driver's settings
# and at its defaults, the ncu launch list, one --set full capture of a paper-scale step at
# A ~ 1000 (t ~ 10) and at t ~ 3000, the regrowth micro and its two captures.
TAG=${1:-r2z}
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/status_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo build=$? >> $OUT/status_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo smoke=$? >> $OUT/status_$TAG.txt
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -rf > $OUT/gpu_tests_$TAG.log 2>&1; echo tests=$? >> $OUT/status_$TAG.txt
fi
timeout 300 python bench.py --steps 20 --warmup 5 > $OUT/bench20_$TAG.json 2> $OUT/bench20_$TAG.err; echo bench20=$? >> $OUT/status_$TAG.txt
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo bench=$? >> $OUT/status_$TAG.txt
CMD="python bench.py --steps 30 --warmup 300 --no-e2e --no-cpu-baseline --no-replay"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s ${NCU_SKIP:-602} -c 60 --csv \
    --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1; echo ncu_launch=$? >> $OUT/status_$TAG.txt
for W in 10 3020; do
  PCMD="python tools/profile_step.py --warmup $W --out $OUT/step_${TAG}_t$W.json"
  timeout 300 $PCMD > $OUT/plain_${TAG}_t$W.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_policy_half|k_prepare_p|k_post" -s $((2 * W)) -c 3 \
      -o $OUT/prof_step_${TAG}_t$W $PCMD > $OUT/ncu_full_${TAG}_t$W.log 2>&1 && \
  python tools/ncu_summary.py $OUT/prof_step_${TAG}_t$W.ncu-rep --step $OUT/step_${TAG}_t$W.json --out $OUT/ncu_summary_${TAG}_t$W.json > /dev/null 2>&1
  echo ncu_full_t$W=$? >> $OUT/status_$TAG.txt
done
if [ "${EXTRA:-1}" = "1" ]; then
timeout 600 python tools/bench_regrowth.py --out $OUT/regrowth_$TAG.json > /dev/null 2> $OUT/regrowth_$TAG.err; echo regrowth=$? >> $OUT/status_$TAG.txt
timeout 900 python bench.py --config large_world --steps 20 --warmup 300 --no-cpu-baseline --no-e2e > $OUT/bench_large_$TAG.json 2> $OUT/bench_large_$TAG.err; echo large=$? >> $OUT/status_$TAG.txt
timeout 900 python bench.py --config ensemble --steps 30 --warmup 20 --no-cpu-baseline --no-e2e > $OUT/bench_ensemble_$TAG.json 2> $OUT/bench_ensemble_$TAG.err; echo ensemble=$? >> $OUT/status_$TAG.txt
fi
cat $OUT/status_$TAG.txt
