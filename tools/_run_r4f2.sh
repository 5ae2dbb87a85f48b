# round-2 (third session, final build) evidence: GPU suite, smoke, default bench, reference arm, launch lists
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4f2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r4f2_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r4f2_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r4f2_pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/r4f2_bench.jsonl 2> gpurun_out/r4f2_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r4f2_bench_ref.jsonl 2> gpurun_out/r4f2_bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r4f2_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu \
  --no-sliced --no-legs --no-pageable > gpurun_out/r4f2_bench_under_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r4f2_launches_bench.csv > gpurun_out/r4f2_launches_bench.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r4f2_syc_slice_launches.csv env NOREF=1 python tools/probe_syc_one.py 12 AUTO > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r4f2_syc_slice_launches.csv > gpurun_out/r4f2_syc_slice_launches.txt
tail -2 gpurun_out/r4f2_smoke.log; tail -3 gpurun_out/r4f2_pytest_gpu.log; head -5 gpurun_out/r4f2_launches_bench.txt; head -8 gpurun_out/r4f2_syc_slice_launches.txt
