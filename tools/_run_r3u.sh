timeout 600 python -m pytest tests/test_gpu_cgemm.py -x -q -k "layout or pair_persistent or variants" 2>&1 | tail -2
timeout 300 python tools/ab_layout.py 2048,16384,64 512,16384,512 2048,4096,32 256,16384,64 2>&1 | cut -c1-250
for i in 1 2; do timeout 600 python bench.py --workload sycamore --steps 3 --warmup 2 2>/dev/null | head -c 200; echo; done
