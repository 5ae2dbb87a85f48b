timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_slicing.py tests/test_gpu_batch_errors.py -x -q > gpurun_out/r2t_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2t_pytest.log
timeout 600 python bench.py --workload sycamore --steps 3 --warmup 2 > gpurun_out/r2t_syc.jsonl 2> gpurun_out/r2t_syc.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2t_syc_slice_launches.csv env NOREF=1 python tools/probe_syc_one.py 12 AUTO > gpurun_out/r2t_syc_one.log 2>&1
python tools/launch_summary.py gpurun_out/r2t_syc_slice_launches.csv > gpurun_out/r2t_syc_slice_summary.txt 2>&1
tail -3 gpurun_out/r2t_pytest.log; head -c 300 gpurun_out/r2t_syc.jsonl; echo; cat gpurun_out/r2t_syc_slice_summary.txt | head -24; tail -3 gpurun_out/r2t_syc_one.log
