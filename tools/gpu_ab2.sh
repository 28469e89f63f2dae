#!/bin/bash
OUT=gpurun_out
for v in libsim libsim_nogreed libsim_notimer libsim_noboth libsim; do
ECO_LIBSIM_OVERRIDE=paper_2302_09334_b200/$v.so timeout 300 python bench.py --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/ab2_$v.json 2>> $OUT/ab2.err
python -c "import json; d=json.loads(open('$OUT/ab2_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,2), {k: round(v*1e3,2) for k,v in d['kernel_ms_per_step'].items()}, {k: round(v,2) for k,v in d['post_phase_us_per_step'].items()})" >> $OUT/ab2.txt
done
