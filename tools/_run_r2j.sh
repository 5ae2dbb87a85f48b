timeout 600 python tools/ab_variant.py TF32TCEC 512,524288,512 512,16384,512 512,8192,1024 2048,16384,64 1024,4096,8192 4096,4096,1024 8192,8192,512 > gpurun_out/r2j_variant.log 2>&1
VARIANTS=wide,wide_persistent timeout 600 python tools/ab_variant.py FP16TCEC 512,16384,512 4096,4096,1024 8192,8192,512 >> gpurun_out/r2j_variant.log 2>&1
cat gpurun_out/r2j_variant.log
