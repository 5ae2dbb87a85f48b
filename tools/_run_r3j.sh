S=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $S --tool racecheck --print-limit 30 --error-exitcode 99 \
    python -m pytest tests/test_gpu_prep.py tests/test_gpu_network.py -q -x -k "prep or skinny_view" -p no:cacheprovider > gpurun_out/r3j_racecheck_prep.log 2>&1
echo "racecheck rc=$?"; tail -4 gpurun_out/r3j_racecheck_prep.log
