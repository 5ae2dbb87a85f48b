set -x
for fl in 1 0; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/gemm4096_f16_flush$fl python tools/prof_gemm.py --n 4096 --mode FP16TCEC --flush $fl --reps 2 > gpurun_out/ncu_f$fl.log 2>&1
done
timeout 400 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:tcec_gemm_kernel --launch-count 1 --csv python tools/prof_gemm.py --n 16384 --mode AUTO --flush 1 --reps 1 > gpurun_out/traffic16384.csv 2>&1
tail -12 gpurun_out/traffic16384.csv
