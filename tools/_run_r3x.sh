timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --launch-skip 0 \
  --log-file gpurun_out/r3x_7x7.csv python tools/probe_7x7.py 16 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r3x_7x7.csv | head -25
