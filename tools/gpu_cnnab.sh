#!/bin/bash
OUT=gpurun_out
: > $OUT/cnnab.txt
timeout 900 python -m pytest tests/test_gpu_cnn.py tests/test_gpu_coloc.py -x -q -s --timeout 600 > $OUT/cnnab_tests.log 2>&1; echo tests=$? >> $OUT/cnnab.txt
for rep in 1 2; do for v in cnnwarp cnnblk; do for C in paper_world_cnn paper_world_coloc; do
  ECO_LIBSIM_OVERRIDE=build_var/libsim_$v.so timeout 300 python bench.py --config $C --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/cnnab_${v}_${C}_$rep.json 2>> $OUT/cnnab.err
  python -c "
import json; d=json.loads(open('$OUT/cnnab_${v}_${C}_$rep.json').read().strip().splitlines()[-1])
print('$v $C', $rep, round(d['ms_per_step']*1e3,2), d.get('graph_kernel_ms_per_step'))" >> $OUT/cnnab.txt 2>&1
done; done; done
cat $OUT/cnnab.txt
