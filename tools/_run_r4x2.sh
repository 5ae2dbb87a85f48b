#!/bin/bash
python -m pytest tests -m gpu -q -k "host or pageable or pipeline or dropin or reference_suite" 2>&1 | tail -2 | tee gpurun_out/r4x2_tests.log
for i in 1 2 3; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-sliced --no-legs 2>/dev/null | grep '^{' | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('value', d['value'], 'e2e', e['value'], 'ratio', round(e['value']/d['value'],4), 'pageable', e.get('pageable',{}).get('value'), 'reruns', e['pipeline']['reruns'], 'sm', d['clocks']['sm_mhz'])" | tee -a gpurun_out/r4x2_tests.log
done
