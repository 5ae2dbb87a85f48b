timeout 300 python tools/ab_small_auto.py 768 1024 1536 2048 4096 > gpurun_out/r2o_small.log 2>&1
VARIANTS=wide,auto,single timeout 300 python tools/ab_variant.py TF32TCEC 1024,1024,1024 128,1024,4096 768,768,768 >> gpurun_out/r2o_small.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2o_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2o_pytest.log
cat gpurun_out/r2o_small.log; tail -3 gpurun_out/r2o_pytest.log
