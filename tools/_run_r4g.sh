#!/bin/bash
# one full ncu capture of the MX=16 skinny column kernel at (16, 2^22, 64) + clocks
SHAPES=16x4194304x64 python tools/bench_skinny.py 2>&1 | tee gpurun_out/r4g_skinny_time.log
SHAPES=16x4194304x64 ncu --set full --clock-control none -k regex:cgemm_skinny_col_kernel -s 2 -c 1 \
    -o gpurun_out/r4g_skinny_col16 python tools/bench_skinny.py > gpurun_out/r4g_ncu.log 2>&1
ncu -i gpurun_out/r4g_skinny_col16.ncu-rep --page raw --csv > gpurun_out/r4g_skinny_col16_raw.csv 2>&1
