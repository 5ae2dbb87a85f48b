#!/bin/bash
python -m pytest tests/test_gpu_stats_adversarial.py -x -q 2>&1 | tail -15 | tee gpurun_out/r4d_tests.log
# per-kernel device times of the skewed (C3) leg
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4d_skewed_launches.csv \
    python bench.py --workload skewed --steps 2 --warmup 1 > gpurun_out/r4d_skewed.log 2>&1
python tools/launch_summary.py gpurun_out/r4d_skewed_launches.csv > gpurun_out/r4d_skewed_launches.txt 2>&1 || true
