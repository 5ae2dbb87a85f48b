VARIANTS=single,pair,wide,wide_persistent timeout 300 python tools/ab_variant.py TF32TCEC 1024,1024,1024 2048,2048,2048 1536,1536,1536 128,1024,4096 256,16384,64 > gpurun_out/r2m_variant.log 2>&1
VARIANTS=single,pair,wide,wide_persistent timeout 300 python tools/ab_variant.py FP16TCEC 1024,1024,1024 2048,2048,2048 >> gpurun_out/r2m_variant.log 2>&1
cat gpurun_out/r2m_variant.log
