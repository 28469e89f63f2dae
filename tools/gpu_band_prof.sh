#!/bin/bash
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_band|k_policy|k_regrow|k_mv" -s ${SKIP:-21760} -c ${COUNT:-136} --csv --log-file gpurun_out/band_launches_${1:-r2j}.csv python tools/profile_band.py --G ${G:-8} --warmup 160 --steps 1 > gpurun_out/band_prof_${1:-r2j}.log 2>&1
tail -3 gpurun_out/band_prof_${1:-r2j}.log
