S=/usr/local/cuda/bin/compute-sanitizer
SEL='tests/test_gpu_kernels.py tests/test_gpu_prep.py tests/test_gpu_cgemm.py tests/test_gpu_network.py tests/test_gpu_batch_errors.py'
DESEL='not full_size and not long_k_kernels and not extreme_aspect and not split_k and not accuracy_uniform and not golden and not 4096 and not 8192 and not all_positive'
rm -f gpurun_out/sanitizer_summary.log
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1500 $S --tool $tool --target-processes all --print-limit 50 --error-exitcode 99 \
    python -m pytest $SEL -q -x -k "$DESEL" -p no:cacheprovider > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_summary.log
  tail -3 gpurun_out/sanitizer_$tool.log >> gpurun_out/sanitizer_summary.log
done
cat gpurun_out/sanitizer_summary.log
