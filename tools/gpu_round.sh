#!/bin/bash
# One GPU job: build, smoke, GPU tests, bench, ncu launch list + one full capture of k_policy.
# Usage (under gpurun): bash tools/gpu_round.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo build=$? > $OUT/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$? >> $OUT/status.txt
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rf > $OUT/gpu_tests.log 2>&1; echo tests=$? >> $OUT/status.txt
fi
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo bench=$? >> $OUT/status.txt
if [ "${SKIP_NCU:-0}" != "1" ]; then
  CMD="python bench.py --steps 30 --warmup 300 --no-e2e --no-cpu-baseline --no-replay"
  timeout 300 $CMD > $OUT/plain_$TAG.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(regrow|policy|post|move|birth|mutate)" \
      -s ${NCU_SKIP:-602} -c 60 --csv --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1
  echo ncu_launch=$? >> $OUT/status.txt
  # one full capture: the graph path's k_post of step W-1, then the instrumented step W's policy and P rows
  W=${PROF_WARMUP:-3020}  # (step W-1 is not a movement-window end)
  PCMD="python tools/profile_step.py --warmup $W --out $OUT/step_$TAG.json"
  timeout 300 $PCMD > $OUT/plain2_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_policy_half|k_prepare_p|k_post" -s $((2 * W)) -c 3 \
      -o $OUT/prof_step_$TAG $PCMD > $OUT/ncu_full_$TAG.log 2>&1 && \
  python tools/ncu_summary.py $OUT/prof_step_$TAG.ncu-rep --step $OUT/step_$TAG.json --out $OUT/ncu_summary_$TAG.json > /dev/null 2>&1
  echo ncu_full=$? >> $OUT/status.txt
fi
cat $OUT/status.txt
if [ "${EXTRA:-0}" = "1" ]; then
  timeout 900 python bench.py --config large_world --steps 20 --warmup 300 --no-cpu-baseline --no-e2e > $OUT/bench_large_$TAG.json 2> $OUT/bench_large_$TAG.err; echo large=$? >> $OUT/status.txt
  timeout 900 python bench.py --config ensemble --steps 30 --warmup 20 --no-cpu-baseline --no-e2e > $OUT/bench_ensemble_$TAG.json 2> $OUT/bench_ensemble_$TAG.err; echo ensemble=$? >> $OUT/status.txt
  timeout 900 python tools/bench_regrowth.py --out $OUT/regrowth_$TAG.json > /dev/null 2> $OUT/regrowth_$TAG.err; echo regrowth=$? >> $OUT/status.txt
  cat $OUT/status.txt
fi
