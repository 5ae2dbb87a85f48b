SHAPES=16x16777216x16,8x33554432x8,32x8388608x16,4x16777216x32,16x4194304x64,8x16777216x8,16x1048576x128,9x100000x77,13x70000x19 timeout 300 python tools/bench_skinny.py > gpurun_out/r2w_skinny.log 2>&1
timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_cgemm.py -x -q -k "skinny or extreme or network or rqc or long_k or fp32" > gpurun_out/r2w_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2w_pytest.log
timeout 600 python bench.py --workload sycamore --steps 3 --warmup 2 > gpurun_out/r2w_syc.jsonl 2> gpurun_out/r2w_syc.err
cat gpurun_out/r2w_skinny.log; tail -2 gpurun_out/r2w_pytest.log; head -c 300 gpurun_out/r2w_syc.jsonl
