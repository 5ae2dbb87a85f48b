#!/bin/bash
# mbarrier try_wait suspend-time hint: A/B on the tensor-bound GEMM (clock under the power cap)
for i in 1 2 3; do
  for lib in paper_2303_08989_b200/libtcec_b200.so abso/libtcec_hint.so; do
    echo -n "$lib: " | tee -a gpurun_out/r4u.log
    TCEC_LIB_PATH=$PWD/$lib VARIANTS=wide timeout 300 python tools/ab_variant.py TF32TCEC 16384,16384,16384 8192,8192,8192 2>&1 | tr '\n' ' ' | tee -a gpurun_out/r4u.log
    echo | tee -a gpurun_out/r4u.log
  done
done
