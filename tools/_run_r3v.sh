S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck; do
timeout 1200 $S --tool $tool --print-limit 20 --error-exitcode 99 python -m pytest tests/test_gpu_cgemm.py -q -x -k "pair_persistent and not all_positive" -p no:cacheprovider > gpurun_out/r3v_$tool.log 2>&1
echo "$tool rc=$?"; tail -2 gpurun_out/r3v_$tool.log
done
