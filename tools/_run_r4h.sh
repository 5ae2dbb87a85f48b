#!/bin/bash
# async-staged skinny column kernel: parity, then A/B vs the register-prefetch kernel
python -m pytest tests/test_gpu_cgemm.py tests/test_gpu_network.py -x -q -k "skinny or fp32 or chain or view or rqc or batch" 2>&1 | tail -3 | tee gpurun_out/r4h_tests.log
for v in 0 1 0 1; do
  echo "== TCEC_SKINNY_ASYNC=$v" | tee -a gpurun_out/r4h_ab.log
  TCEC_SKINNY_ASYNC=$v SHAPES=16x4194304x64,16x16777216x16,8x16777216x8,8x33554432x8,16x16777216x8,32x8388608x16 python tools/bench_skinny.py 2>&1 | tee -a gpurun_out/r4h_ab.log
  TCEC_SKINNY_ASYNC=$v python tools/bench_skinny_view.py 24 6 4 2>&1 | tail -2 | tee -a gpurun_out/r4h_ab.log
done
for v in 0 1; do
  echo "== sycamore TCEC_SKINNY_ASYNC=$v" | tee -a gpurun_out/r4h_ab.log
  TCEC_SKINNY_ASYNC=$v timeout 600 python bench.py --workload sycamore --steps 3 --warmup 1 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['unit'], d.get('ms_per_step'))" | tee -a gpurun_out/r4h_ab.log
done
