VARIANTS=auto,single,pair,wide timeout 300 python tools/ab_variant.py TF32TCEC 1024,1024,1024 128,1024,4096 512,512,4096 256,256,65536 1024,512,2048 768,768,768 > gpurun_out/r2n_variant.log 2>&1
cat gpurun_out/r2n_variant.log
