#!/bin/bash
for cfg in "0 4" "1 2" "1 3" "1 4"; do
  set -- $cfg
  TCEC_SKINNY_ASYNC=$1 TCEC_SKINNY_VSTAGES=$2 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r4j_syc_$1_$2.csv env NOREF=1 python tools/probe_syc_one.py 12 AUTO > /dev/null 2>&1
  echo "== async=$1 vstages=$2" >> gpurun_out/r4j_summary.txt
  python tools/launch_summary.py gpurun_out/r4j_syc_$1_$2.csv | grep -E "skinny_col|TOTAL" >> gpurun_out/r4j_summary.txt
done
