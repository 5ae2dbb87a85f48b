#!/bin/bash
# flush-interval cost on the current wide kernel (diagnostic; flush != 1 changes the numerics)
NS=8192,16384 MODES=TF32TCEC,TF32TC python tools/flush_sweep.py 2>&1 | tee gpurun_out/r4b_flush.log
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv | tee -a gpurun_out/r4b_flush.log
