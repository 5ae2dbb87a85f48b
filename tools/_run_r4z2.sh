#!/bin/bash
# racecheck (shared-memory hazards) over the kernels changed this session, to completion
S=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $S --tool racecheck --target-processes all --print-limit 50 --error-exitcode 99 \
  python -m pytest tests/test_gpu_stats_adversarial.py tests/test_gpu_cgemm.py tests/test_gpu_network.py -q -x \
  -k "adversarial or sizes_and_offsets or dispatch_decision_adversarial or skinny_kernels_bit_exact or skinny_view" -p no:cacheprovider \
  > gpurun_out/r4z2_racecheck.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/r4z2_racecheck.log
tail -4 gpurun_out/r4z2_racecheck.log
