set -x
SHAPES=16x16777216x16,8x33554432x8,32x8388608x16,16777216x8x8,4194304x16x64,4194304x32x8,16777216x16x16,67108864x2x2,8388608x8x8,2097152x16x32,16777216x4x4 timeout 300 python tools/bench_skinny.py > gpurun_out/r2h_skinny.log 2>&1
timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_cgemm.py -x -q -k "skinny or extreme or network or rqc or long_k" > gpurun_out/r2h_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2h_pytest.log
timeout 600 python bench.py --workload sycamore --steps 3 --warmup 2 > gpurun_out/r2h_syc.jsonl 2> gpurun_out/r2h_syc.err
cat gpurun_out/r2h_skinny.log; tail -2 gpurun_out/r2h_pytest.log; head -c 300 gpurun_out/r2h_syc.jsonl
echo "--- previous build (row kernel not persistent)"
SHAPES=16777216x8x8,4194304x16x64,4194304x32x8,16777216x16x16,67108864x2x2,8388608x8x8,2097152x16x32,16777216x4x4 TCEC_LIB_PATH=oldlib/libtcec_prev.so timeout 300 python tools/bench_skinny.py
