#!/bin/bash
python tools/ab_env_skewed.py TCEC_STATS_KEEP 0 1 2>&1 | tee gpurun_out/r4e_ab_keep.log
