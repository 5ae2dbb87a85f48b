set -x
timeout 600 python bench.py --workload sycamore --steps 2 --warmup 1 > gpurun_out/r2c_syc_bench.jsonl 2> gpurun_out/r2c_syc_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2c_syc_slice_launches.csv python tools/probe_syc_one.py 12 AUTO > gpurun_out/r2c_syc_one.log 2>&1
python tools/launch_summary.py gpurun_out/r2c_syc_slice_launches.csv > gpurun_out/r2c_syc_slice_summary.txt 2>&1
timeout 900 python tools/step_profile.py 12 > gpurun_out/r2c_step_profile.txt 2>&1
head -30 gpurun_out/r2c_syc_slice_summary.txt; head -30 gpurun_out/r2c_step_profile.txt
