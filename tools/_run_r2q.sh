REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2q_c3_launches.csv python tools/ab_layout.py 512,16384,512 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2q_c3_launches.csv | head -12
timeout 300 python tools/ab_layout.py > gpurun_out/r2q_ab_layout.log 2>&1
timeout 300 python tools/ab_small_auto.py 1024 2048 4096 >> gpurun_out/r2q_ab_layout.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dispatch.py tests/test_gpu_headline.py -x -q > gpurun_out/r2q_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2q_pytest.log
cat gpurun_out/r2q_ab_layout.log; tail -2 gpurun_out/r2q_pytest.log
