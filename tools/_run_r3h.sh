SHAPES=16x16777216x16 timeout 600 ncu --set full --clock-control none -k regex:skinny_col --launch-skip 1 --launch-count 1 -o gpurun_out/r3h_col16 -f python tools/bench_skinny.py > /dev/null 2>&1
ls gpurun_out/r3h_col16.ncu-rep
