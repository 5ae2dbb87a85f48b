timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dispatch.py tests/test_gpu_headline.py -q -x > gpurun_out/t_stats.log 2>&1
echo "rc=$?" >> gpurun_out/t_stats.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_skewed.py 512,16384,512 1024,4096,8192 > gpurun_out/r02_skewed_launches2.csv 2>&1
