#!/bin/bash
# DRAM traffic and time of the 16384^3 TF32 GEMM: one-tile-per-cluster wide vs persistent widep
for v in wide wide_persistent; do
  echo "== $v" >> gpurun_out/r4m_traffic.txt
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none \
    -k regex:tcec_gemm_wide --launch-count 1 --csv python tools/prof_gemm.py --n 16384 --mode AUTO --ref-inputs --reps 1 --variant $v 2>&1 \
    | grep -E "dram__bytes|duration|lts__t_bytes" | awk -F'","' '{print $13, $15}' >> gpurun_out/r4m_traffic.txt
done
VARIANTS=wide,wide_persistent python tools/ab_variant.py TF32TCEC 16384,16384,16384 8192,8192,8192 2>&1 | tee -a gpurun_out/r4m_traffic.txt
VARIANTS=wide,wide_persistent python tools/ab_variant.py TF32TCEC 16384,16384,16384 2>&1 | tee -a gpurun_out/r4m_traffic.txt
