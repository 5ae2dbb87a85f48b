timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r3t_pytest.log; tail -3 gpurun_out/r3t_pytest.log
grep -E "FAILED|Error" gpurun_out/r3t_pytest.log | head
