set -x
timeout 900 python -m pytest tests/test_gpu_prep.py tests/test_gpu_cgemm.py -x -q > gpurun_out/r2a_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2a_pytest.log
timeout 600 python tools/ab_layout.py > gpurun_out/r2a_ab_layout.log 2>&1
tail -3 gpurun_out/r2a_pytest.log; cat gpurun_out/r2a_ab_layout.log
