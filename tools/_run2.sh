M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second
for v in wide_mc wide; do
  TCEC_VARIANT=$v timeout 600 ncu --metrics $M --clock-control none -k regex:tcec_gemm_wide --launch-count 1 --csv \
    python tools/prof_gemm.py --n 16384 --mode AUTO --reps 1 --ref-inputs --variant $v > gpurun_out/r02_traffic16384_tf32_$v.csv 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_skewed.py > gpurun_out/r02_skewed_launches.csv 2>&1
