VARIANTS=wide timeout 600 ncu --set full --clock-control none -k regex:tcec_gemm_wide_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/r3q_wide_512x524288 -f python tools/ab_variant.py TF32TCEC 512,524288,512 > gpurun_out/r3q.log 2>&1
VARIANTS=wide_persistent timeout 600 ncu --set full --clock-control none -k regex:widep --launch-skip 1 --launch-count 1 -o gpurun_out/r3q_widep_512x524288 -f python tools/ab_variant.py TF32TCEC 512,524288,512 >> gpurun_out/r3q.log 2>&1
ls gpurun_out/r3q*
