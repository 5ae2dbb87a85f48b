#!/bin/bash
python tools/ab_env_skewed.py TCEC_STATS_F4 4 8 16 2>&1 | head -8 | tee gpurun_out/r4w.log
python tools/ab_env_skewed.py TCEC_STATS_F4 4 16 2>&1 | tail -2 | tee -a gpurun_out/r4w.log
