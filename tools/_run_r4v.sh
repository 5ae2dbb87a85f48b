#!/bin/bash
python -m pytest tests/test_gpu_cgemm.py -q -k skinny_kernels_bit_exact 2>&1 | tail -3 | tee gpurun_out/r4v.log
TCEC_SKINNY_ASYNC=0 python -m pytest tests/test_gpu_cgemm.py -q -k skinny_kernels_bit_exact 2>&1 | tail -2 | tee -a gpurun_out/r4v.log
