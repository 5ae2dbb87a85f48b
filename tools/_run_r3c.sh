for v in 1 0; do TCEC_VIEW_GATHER=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3c_$v.csv python tools/bench_skinny_view.py 28 6 4 1 > /dev/null 2>&1; echo "== view=$v"; python tools/launch_summary.py gpurun_out/r3c_$v.csv | head -3; done
SHAPES=16777216x8x8,4194304x16x64,4194304x32x8,16777216x16x16,67108864x2x2,8388608x8x8 timeout 300 python tools/bench_skinny.py
timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_cgemm.py -x -q -k "skinny or extreme or network or rqc or long_k or fp32" > gpurun_out/r3c_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3c_pytest.log; tail -2 gpurun_out/r3c_pytest.log
timeout 600 python bench.py --workload sycamore --steps 3 --warmup 2 > gpurun_out/r3c_syc.jsonl 2> gpurun_out/r3c_syc.err; head -c 300 gpurun_out/r3c_syc.jsonl
