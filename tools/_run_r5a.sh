#!/bin/bash
# raster group of the default wide kernel on the TF32 headline shape
for g in ${GS:-4 3 5 6 4 3 5 6}; do
  echo -n "group_m=$g: " | tee -a gpurun_out/r5a.log
  TCEC_GROUP_M=$g VARIANTS=wide timeout 300 python tools/ab_variant.py TF32TCEC 16384,16384,16384 2>&1 | tail -1 | tee -a gpurun_out/r5a.log
done
