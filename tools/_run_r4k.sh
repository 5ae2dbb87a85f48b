#!/bin/bash
python -m pytest tests/test_gpu_cgemm.py tests/test_gpu_network.py tests/test_gpu_slicing.py -x -q 2>&1 | tail -3 | tee gpurun_out/r4k_tests.log
for v in 0 1; do
  TCEC_SKINNY_ASYNC=$v ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r4k_syc_$v.csv env NOREF=1 python tools/probe_syc_one.py 12 AUTO > /dev/null 2>&1
  echo "== async=$v" >> gpurun_out/r4k_summary.txt
  python tools/launch_summary.py gpurun_out/r4k_syc_$v.csv | grep -E "skinny_col|TOTAL" >> gpurun_out/r4k_summary.txt
done
for v in 0 1 0 1; do
  echo "== TCEC_SKINNY_ASYNC=$v" | tee -a gpurun_out/r4k_ab.log
  TCEC_SKINNY_ASYNC=$v SHAPES=16x4194304x64,16x16777216x16,8x16777216x8,8x33554432x8,16x16777216x8,32x8388608x16 python tools/bench_skinny.py 2>&1 | tee -a gpurun_out/r4k_ab.log
  TCEC_SKINNY_ASYNC=$v timeout 600 python bench.py --workload sycamore --steps 3 --warmup 1 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['unit'], d.get('ms_per_step'), d.get('clocks'))" | tee -a gpurun_out/r4k_ab.log
done
