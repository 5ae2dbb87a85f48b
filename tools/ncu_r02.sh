# ncu evidence for the round-2 headline (run under gpurun, one GPU):
#  1. launch list of the default bench command (per-launch times, cold/serialised)
#  2. DRAM traffic of the wide kernel at n=16384 on the reference inputs (TF32 path,
#     the AUTO decision) and forced FP16TCEC (f16 path) -> bench roofline.traffic
#  3. one --set full capture of the wide kernel's TF32 path at n=4096
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu \
  --no-sliced --no-legs --no-pageable > gpurun_out/r02_bench_under_ncu.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second
timeout 600 ncu --metrics $M --clock-control none -k regex:tcec_gemm_wide --launch-count 1 --csv \
  python tools/prof_gemm.py --n 16384 --mode AUTO --reps 1 --ref-inputs > gpurun_out/r02_traffic16384_tf32.csv 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:tcec_gemm_wide --launch-count 1 --csv \
  python tools/prof_gemm.py --n 16384 --mode FP16TCEC --reps 1 > gpurun_out/r02_traffic16384_f16.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm_wide \
  --launch-skip 1 --launch-count 1 -o gpurun_out/r02_wide4096_tf32 -f \
  python tools/prof_gemm.py --n 4096 --mode TF32TCEC --reps 2 > gpurun_out/r02_ncu_full.log 2>&1
tail -6 gpurun_out/r02_traffic16384_tf32.csv gpurun_out/r02_traffic16384_f16.csv
