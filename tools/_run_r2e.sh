set -x
timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_slicing.py tests/test_gpu_batch_errors.py -x -q > gpurun_out/r2e_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2e_pytest.log
SHAPES=16x16777216x16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:skinny_col \
  --launch-skip 1 --launch-count 1 -o gpurun_out/r2e_skinny_col16 -f python tools/bench_skinny.py > gpurun_out/r2e_ncu_skinny.log 2>&1
SHAPES=16x16777216x16,8x33554432x8,32x8388608x16,16777216x8x8 timeout 300 python tools/bench_skinny.py > gpurun_out/r2e_skinny.log 2>&1
tail -3 gpurun_out/r2e_pytest.log; cat gpurun_out/r2e_skinny.log; tail -3 gpurun_out/r2e_ncu_skinny.log
