VARIANTS=wide_persistent timeout 600 ncu --set full --import-source on --clock-control none -k regex:widep --launch-skip 1 --launch-count 1 -o gpurun_out/r3b_widep_smallk -f python tools/ab_variant.py TF32TCEC 2048,16384,64 > gpurun_out/r3b.log 2>&1
tail -2 gpurun_out/r3b.log
