#!/bin/bash
# K sweep of the TF32TCEC step shape family: per-tile overhead vs k
export VARIANTS=wide,wide_persistent,pair_persistent
python tools/ab_variant.py TF32TCEC 512,131072,256 512,131072,512 512,131072,1024 512,131072,2048 512,131072,4096 512,65536,8192 2>&1 | tee gpurun_out/r4a_ksweep.log
python tools/ab_variant.py FP16TCEC 512,131072,512 512,131072,1024 512,131072,2048 512,65536,8192 2>&1 | tee -a gpurun_out/r4a_ksweep.log
