timeout 900 python -m pytest tests/test_gpu_prep.py tests/test_gpu_network.py -x -q -k "prep or view or rqc or network" > gpurun_out/r3d_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3d_pytest.log; tail -2 gpurun_out/r3d_pytest.log
timeout 300 python tools/ab_layout.py 512,16384,512 512,8192,1024 512,524288,512 16384,16384,16384 2>&1 | cut -c1-250
timeout 600 python bench.py --workload sycamore --steps 3 --warmup 2 > gpurun_out/r3d_syc.jsonl 2> gpurun_out/r3d_syc.err; head -c 300 gpurun_out/r3d_syc.jsonl
