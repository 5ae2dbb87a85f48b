for sp in 0 1; do echo "SPLIT2=$sp"; TCEC_SKINNY_SPLIT2=$sp SHAPES=16x16777216x16,32x8388608x16,16x4194304x64,9x2000000x16,13x70000x19,16x1048576x128 timeout 300 python tools/bench_skinny.py; done
timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_cgemm.py -x -q -k "skinny or extreme or network or rqc or long_k or fp32" 2>&1 | tail -2
for sp in 0 1; do TCEC_SKINNY_SPLIT2=$sp timeout 600 python bench.py --workload sycamore --steps 3 --warmup 2 2>/dev/null | head -c 260; echo; done
