# session re-entry check: GPU suite + default bench + step profile of C3 shapes
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2s_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2s_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2s_bench.jsonl 2> gpurun_out/r2s_bench.err
echo "bench rc=$?"
timeout 300 python tools/prof_skewed.py > gpurun_out/r2s_skewed.log 2>&1
tail -3 gpurun_out/r2s_pytest_gpu.log
