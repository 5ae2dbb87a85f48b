timeout 900 python -m pytest tests/test_gpu_dispatch.py tests/test_gpu_kernels.py tests/test_gpu_headline.py tests/test_gpu_cgemm.py -x -q > gpurun_out/r3m_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r3m_pytest.log; tail -2 gpurun_out/r3m_pytest.log
for f in 0 1; do echo "TCEC_PREAMBLE=$f"; TCEC_PREAMBLE=$f timeout 300 python tools/ab_layout.py 2048,16384,64 2048,4096,32 256,16384,64 128,1024,4096 512,16384,512 512,8192,1024 2>&1 | cut -c1-140; TCEC_PREAMBLE=$f timeout 300 python tools/ab_small_auto.py 768 1024 1536 2048; done
