S=/usr/local/cuda/bin/compute-sanitizer
SEL='tests/test_gpu_prep.py tests/test_gpu_network.py'
for tool in racecheck memcheck; do
  timeout 1500 $S --tool $tool --target-processes all --print-limit 30 --error-exitcode 99 \
    python -m pytest $SEL -q -x -k "not 7x7 and not sycamore and not hyper" -p no:cacheprovider > gpurun_out/r3i_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r3i_sanitizer_$tool.log
done
