#!/bin/bash
# why is the persistent wide kernel slower in steady state? ncu full on 8192^3 TF32 for both
for v in wide wide_persistent; do
  timeout 900 ncu --set full --clock-control none -k regex:tcec_gemm_wide --launch-count 1 \
    -o gpurun_out/r4t_$v python tools/prof_gemm.py --n 8192 --mode TF32TCEC --reps 1 --variant $v > gpurun_out/r4t_$v.log 2>&1
  ncu -i gpurun_out/r4t_$v.ncu-rep --page raw --csv > gpurun_out/r4t_${v}_raw.csv 2>&1
  rm -f gpurun_out/r4t_$v.ncu-rep
done
