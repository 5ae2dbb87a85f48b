#!/bin/bash
for v in 1 0; do
  echo "== TCEC_HOST_SPEC_TF32=$v" | tee -a gpurun_out/r5k.log
  TCEC_HOST_SPEC_TF32=$v timeout 900 python tools/ab_host_e2e.py 8192 10240 12288 14336 16384 2>&1 | tail -5 | tee -a gpurun_out/r5k.log
done
python -m pytest tests -m gpu -q -k "host or pageable or pipeline or dropin" 2>&1 | tail -2 | tee -a gpurun_out/r5k.log
