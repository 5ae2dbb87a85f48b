#!/bin/bash
python -m pytest tests -m gpu -q -k "host or pageable or pipeline or dropin" 2>&1 | tail -2 | tee gpurun_out/r5l.log
timeout 900 python tools/probe_host_shapes.py 2>&1 | tail -6 | tee -a gpurun_out/r5l.log
timeout 900 python tools/ab_host_e2e.py 8192 10240 12288 14336 16384 2>&1 | tail -5 | tee -a gpurun_out/r5l.log
