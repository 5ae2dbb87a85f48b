timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r3s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r3s_pytest.log; tail -3 gpurun_out/r3s_pytest.log
timeout 300 python tools/ab_layout.py 2048,16384,64 512,16384,512 512,8192,1024 2048,4096,32 256,16384,64 128,1024,4096 1024,4096,8192 2>&1 | cut -c1-150
timeout 600 python bench.py --workload skewed --steps 5 --warmup 3 2>/dev/null | head -c 200; echo
timeout 600 python bench.py --workload sycamore --steps 3 --warmup 2 2>/dev/null | head -c 200; echo
