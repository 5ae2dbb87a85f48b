#!/bin/bash
# k-progress throttle in the persistent wide kernel: bit identity, time and DRAM bytes at 16384^3 TF32
TCEC_THROTTLE=48 TCEC_GROUP_M_P=8 timeout 300 python tools/check_widep_throttle.py 2>&1 | tail -4 | tee gpurun_out/r4s.log
for cfg in "0 16" "64 16" "64 8" "32 8" "128 8" "16 8"; do
  set -- $cfg
  echo -n "throttle=$1 group=$2: " | tee -a gpurun_out/r4s.log
  TCEC_THROTTLE=$1 TCEC_GROUP_M_P=$2 VARIANTS=wide,wide_persistent timeout 300 python tools/ab_variant.py TF32TCEC 16384,16384,16384 2>&1 | tail -1 | tee -a gpurun_out/r4s.log
done
for cfg in "64 8" "32 8"; do
  set -- $cfg
  echo "== ncu throttle=$1 group=$2" >> gpurun_out/r4s.log
  TCEC_THROTTLE=$1 TCEC_GROUP_M_P=$2 timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none \
    -k regex:tcec_gemm_wide --launch-count 1 --csv python tools/prof_gemm.py --n 16384 --mode AUTO --ref-inputs --reps 1 --variant wide_persistent 2>&1 \
    | grep -E "dram__bytes|duration" | awk -F'","' '{print $13, $15}' >> gpurun_out/r4s.log
done
