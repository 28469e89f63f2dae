#!/bin/bash
# A/B of library variants in build_var/ on the 64-world ensemble (configs[4]): bench.py
# --config ensemble --steps 30 --warmup 20 per variant.  Usage: bash tools/gpu_ab_ens.sh v1 v2 ...
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/ab_ens.txt
for v in "$@"; do
  ECO_LIBSIM_OVERRIDE=build_var/libsim_$v.so timeout 600 python bench.py --config ensemble --steps 30 --warmup 20 --no-cpu-baseline --no-e2e > $OUT/ens_$v.json 2>> $OUT/ab_ens.err
  python -c "
import json; d=json.loads(open('$OUT/ens_$v.json').read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step']*1e3,2), {k: round(x, 1) for k, x in d['post_phase_us_per_step'].items()}, d.get('graph_kernel_ms_per_step'), d.get('replay_identical'))" >> $OUT/ab_ens.txt 2>&1
done
cat $OUT/ab_ens.txt
