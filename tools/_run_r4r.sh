#!/bin/bash
# sanitizer pass over the kernels changed in this session: statistics (selection in
# stats2's last block), cp.async skinny column kernels (plain + gathered views),
# dispatch decisions
S=/usr/local/cuda/bin/compute-sanitizer
SEL='tests/test_gpu_stats_adversarial.py tests/test_gpu_kernels.py tests/test_gpu_dispatch.py tests/test_gpu_network.py'
DESEL='not golden and not 4096 and not 8192 and not host_pipeline and not full_size'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $S --tool $tool --target-processes all --print-limit 50 --error-exitcode 99 \
    python -m pytest $SEL -q -x -k "$DESEL" -p no:cacheprovider > gpurun_out/r4r_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r4r_sanitizer_summary.log
  tail -3 gpurun_out/r4r_sanitizer_$tool.log >> gpurun_out/r4r_sanitizer_summary.log
done
