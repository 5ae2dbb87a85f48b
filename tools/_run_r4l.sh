#!/bin/bash
# row kernel f32x2 chains: parity, then A/B against the previous library (abso/libtcec_prev.so)
python -m pytest tests/test_gpu_cgemm.py tests/test_gpu_network.py -x -q -k "skinny or fp32 or view or rqc or chain" 2>&1 | tail -2 | tee gpurun_out/r4l_tests.log
for lib in abso/libtcec_prev.so paper_2303_08989_b200/libtcec_b200.so abso/libtcec_prev.so paper_2303_08989_b200/libtcec_b200.so; do
  echo "== $lib" | tee -a gpurun_out/r4l_ab.log
  TCEC_LIB_PATH=$PWD/$lib SHAPES=16777216x8x8,4194304x16x64,4194304x32x8,2097152x16x32,1048576x16x16,8388608x8x8,4194304x8x16 python tools/bench_skinny.py 2>&1 | tee -a gpurun_out/r4l_ab.log
done
for lib in abso/libtcec_prev.so paper_2303_08989_b200/libtcec_b200.so; do
  TCEC_LIB_PATH=$PWD/$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r4l_syc.csv env NOREF=1 python tools/probe_syc_one.py 12 AUTO > /dev/null 2>&1
  echo "== $lib" >> gpurun_out/r4l_summary.txt
  python tools/launch_summary.py gpurun_out/r4l_syc.csv | grep -E "skinny_row|TOTAL" >> gpurun_out/r4l_summary.txt
done
