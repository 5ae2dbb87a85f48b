set -x
SHAPES=16777216x8x8,4194304x16x64,4194304x32x8,16777216x16x16,67108864x2x2,8388608x8x8,2097152x16x32,16777216x4x4 timeout 300 python tools/bench_skinny.py > gpurun_out/r2i_skinny.log 2>&1
timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_cgemm.py -x -q -k "skinny or extreme or network or rqc or long_k" > gpurun_out/r2i_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2i_pytest.log
timeout 600 python bench.py --workload sycamore --steps 3 --warmup 2 > gpurun_out/r2i_syc.jsonl 2> gpurun_out/r2i_syc.err
SHAPES=16x16777216x16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:skinny_col \
  --launch-skip 1 --launch-count 1 -o gpurun_out/r2i_skinny_col16 -f python tools/bench_skinny.py > gpurun_out/r2i_ncu_skinny.log 2>&1
cat gpurun_out/r2i_skinny.log; tail -2 gpurun_out/r2i_pytest.log; head -c 300 gpurun_out/r2i_syc.jsonl
