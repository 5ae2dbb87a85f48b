#!/bin/bash
SHAPES=4194304x16x64 ncu --set full --clock-control none -k regex:cgemm_skinny_row_kernel -s 2 -c 1 \
    -o gpurun_out/r4q_row16 python tools/bench_skinny.py > gpurun_out/r4q_ncu.log 2>&1
ncu -i gpurun_out/r4q_row16.ncu-rep --page raw --csv > gpurun_out/r4q_row16_raw.csv 2>&1
rm -f gpurun_out/r4q_row16.ncu-rep
