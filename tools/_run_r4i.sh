#!/bin/bash
# Sycamore slice per-kernel times with / without the async column kernel, + the leg twice per arm
for v in 0 1; do
  TCEC_SKINNY_ASYNC=$v ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r4i_syc_launches_$v.csv env NOREF=1 python tools/probe_syc_one.py 12 AUTO > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/r4i_syc_launches_$v.csv > gpurun_out/r4i_syc_launches_$v.txt
done
for v in 0 1 0 1; do
  echo "== TCEC_SKINNY_ASYNC=$v" | tee -a gpurun_out/r4i_ab.log
  TCEC_SKINNY_ASYNC=$v python tools/bench_skinny_view.py 24 6 4 2>&1 | tail -1 | tee -a gpurun_out/r4i_ab.log
  TCEC_SKINNY_ASYNC=$v timeout 600 python bench.py --workload sycamore --steps 3 --warmup 1 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['unit'], d.get('ms_per_step'), d.get('clocks'))" | tee -a gpurun_out/r4i_ab.log
done
