# ncu evidence for the headline kernel (run under gpurun, one GPU):
#  1. launch list of the default bench command (per-launch times, cold/serialised)
#  2. one --set full capture of the wide f16 TCEC kernel at n=4096
#  3. DRAM traffic of the wide f16 kernel at n=16384 (bench roofline.traffic)
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu \
  > gpurun_out/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm_wide \
  --launch-skip 1 --launch-count 1 -o gpurun_out/wide4096_f16 -f \
  python tools/prof_gemm.py --n 4096 --mode AUTO --reps 2 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
  --clock-control none -k regex:tcec_gemm_wide --launch-count 1 --csv \
  python tools/prof_gemm.py --n 16384 --mode AUTO --reps 1 > gpurun_out/traffic16384.csv 2>&1
tail -12 gpurun_out/traffic16384.csv
