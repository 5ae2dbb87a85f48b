set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_pytest.log
for f in 0 1; do echo "TCEC_PREAMBLE=$f"; TCEC_PREAMBLE=$f timeout 600 python tools/ab_layout.py; done > gpurun_out/r2b_ab_preamble.log 2>&1
for f in 0 1; do echo "TCEC_PREAMBLE=$f"; TCEC_PREAMBLE=$f REPS=3 timeout 600 python tools/ab_layout.py 4096,4096,4096 16384,16384,16384 2048,2048,2048 1024,1024,1024; done >> gpurun_out/r2b_ab_preamble.log 2>&1
tail -3 gpurun_out/r2b_pytest.log; cat gpurun_out/r2b_ab_preamble.log
