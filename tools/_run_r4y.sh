#!/bin/bash
nproc | tee gpurun_out/r4y.log
for c in 16 12 16 12; do
  TCEC_HOST_CHUNKS=$c timeout 600 python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-sliced --no-legs 2>/dev/null | grep '^{' | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('chunks=$c value', d['value'], 'e2e', e['value'], 'ratio', round(e['value']/d['value'],4), 'pageable', e.get('pageable',{}).get('value'), 'sm', d['clocks']['sm_mhz'])" | tee -a gpurun_out/r4y.log
done
