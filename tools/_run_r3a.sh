timeout 900 python -m pytest tests/test_gpu_cgemm.py tests/test_gpu_dispatch.py -x -q > gpurun_out/r3a_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3a_pytest.log; tail -3 gpurun_out/r3a_pytest.log
for t in 0 1; do echo "TCEC_TMA_STORE=$t"; TCEC_TMA_STORE=$t VARIANTS=wide_persistent,auto timeout 300 python tools/ab_variant.py TF32TCEC 2048,16384,64 256,16384,64 2048,4096,32 512,16384,512 4096,4096,256 8192,8192,128; done
for t in 0 1; do echo "TCEC_TMA_STORE=$t"; TCEC_TMA_STORE=$t VARIANTS=wide_persistent timeout 300 python tools/ab_variant.py FP16TCEC 2048,16384,64 8192,8192,128; done
