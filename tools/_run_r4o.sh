#!/bin/bash
# host pipeline knobs: A row chunks x B front parts -> e2e / device value
for cfg in ${CFGS:-"16 2" "24 2" "32 2" "16 2" "24 2" "32 2" "24 3"}; do
  set -- $cfg
  TCEC_HOST_CHUNKS=$1 TCEC_HOST_BFRONT=$2 timeout 600 python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-sliced --no-legs --no-pageable 2>/dev/null | grep '^{' | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('chunks=$1 bfront=$2 value', d['value'], 'e2e', e['value'], 'ratio', round(e['value']/d['value'],4), 'reruns', e['pipeline']['reruns'], 'sm', d['clocks']['sm_mhz'])" | tee -a gpurun_out/r4o_host_knobs2.log
done
