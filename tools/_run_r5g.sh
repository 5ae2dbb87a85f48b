#!/bin/bash
python -m pytest tests -m gpu -q -k "profile or dispatch or graph or skinny_kernels" 2>&1 | tail -2 | tee gpurun_out/r5g.log
timeout 600 python bench.py --workload skewed --steps 20 --warmup 3 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('leg', d['value'])
for s in d['shapes']: print(s['m'], s['n'], s['k'], s['ms'], s['floor_frac_hbm'], s.get('stages_ms'))
" | tee -a gpurun_out/r5g.log
