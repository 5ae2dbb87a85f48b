REPS=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:stats2 --launch-skip 2 --launch-count 1 -o gpurun_out/r2p_stats2 -f python tools/ab_layout.py 512,16384,512 > /dev/null 2>&1
REPS=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:prep_bx --launch-skip 2 --launch-count 1 -o gpurun_out/r2p_prep_bx -f python tools/ab_layout.py 512,16384,512 > /dev/null 2>&1
ls -la gpurun_out/r2p*
