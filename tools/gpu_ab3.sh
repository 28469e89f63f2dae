#!/bin/bash
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 900 -rf -x -k "paper_world or tiny or greed or checks or graph_equals" > $OUT/ab3_tests.log 2>&1; echo tests=$? >> $OUT/ab3_tests.log
timeout 300 python bench.py --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/ab3_b2000.json 2>> $OUT/ab3.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/ab3_b20.json 2>> $OUT/ab3.err
for f in ab3_b2000 ab3_b20; do python -c "import json; d=json.loads(open('$OUT/$f.json').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step']*1e3,2), {k: round(v,2) for k,v in d['post_phase_us_per_step'].items()})" >> $OUT/ab3.txt; done
