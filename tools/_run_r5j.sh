#!/bin/bash
for v in 1024 256 1024 256; do
  echo -n "minrows=$v " | tee -a gpurun_out/r5j.log
  TCEC_HOST_MINROWS=$v timeout 600 python tools/ab_host_e2e.py 8192 12288 2>&1 | tr '\n' ' ' | tee -a gpurun_out/r5j.log
  echo | tee -a gpurun_out/r5j.log
done
python -m pytest tests -m gpu -q -k "host or pageable or pipeline" 2>&1 | tail -2 | tee -a gpurun_out/r5j.log
