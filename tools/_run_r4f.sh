#!/bin/bash
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/r4f_pytest.log
python tools/ab_env_skewed.py TCEC_STATS_KEEP 0 1 2>&1 | tee gpurun_out/r4f_ab_keep.log
