#!/bin/bash
timeout 900 ncu --set full --clock-control none -k regex:tcec_gemm_pairp --launch-count 1 -s 2 \
  -o gpurun_out/r5f_pairp python tools/prof_gemm.py --m 2048 --n 16384 --k 64 --mode TF32TCEC --reps 3 > gpurun_out/r5f.log 2>&1
ncu -i gpurun_out/r5f_pairp.ncu-rep --page raw --csv > gpurun_out/r5f_pairp_raw.csv 2>&1
ncu -i gpurun_out/r5f_pairp.ncu-rep --page source --csv --print-source sass > gpurun_out/r5f_pairp_source.csv 2>&1
rm -f gpurun_out/r5f_pairp.ncu-rep
