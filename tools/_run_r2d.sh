set -x
timeout 900 python -m pytest tests/test_gpu_network.py tests/test_gpu_slicing.py tests/test_gpu_batch_errors.py -x -q > gpurun_out/r2d_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2d_pytest.log
for f in 0 1; do TCEC_VIEW_GATHER=$f timeout 600 python bench.py --workload sycamore --steps 3 --warmup 2 > gpurun_out/r2d_syc_view$f.jsonl 2> gpurun_out/r2d_syc_view$f.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2d_syc_slice_launches.csv python tools/probe_syc_one.py 12 AUTO > gpurun_out/r2d_syc_one.log 2>&1
python tools/launch_summary.py gpurun_out/r2d_syc_slice_launches.csv > gpurun_out/r2d_syc_slice_summary.txt 2>&1
tail -3 gpurun_out/r2d_pytest.log; head -c 400 gpurun_out/r2d_syc_view0.jsonl; echo; head -c 400 gpurun_out/r2d_syc_view1.jsonl; echo; cat gpurun_out/r2d_syc_slice_summary.txt; cat gpurun_out/r2d_syc_one.log | tail -3
