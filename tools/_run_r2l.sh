for kb in 32 16 8 4; do echo "TCEC_SPLIT_MINKB=$kb"; TCEC_SPLIT_MINKB=$kb timeout 300 python tools/ab_small_auto.py 1024 2048 4096; done > gpurun_out/r2l_split.log 2>&1
echo "single:" >> gpurun_out/r2l_split.log
cat gpurun_out/r2l_split.log
