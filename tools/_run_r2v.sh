for v in 1 0; do
  TCEC_VIEW_GATHER=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2v_$v.csv python tools/bench_skinny_view.py 28 6 4 1 > /dev/null 2>&1
  echo "== view=$v"; python tools/launch_summary.py gpurun_out/r2v_$v.csv | head -3
  TCEC_VIEW_GATHER=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2v_c$v.csv python tools/bench_skinny_view.py 28 4 4 0 > /dev/null 2>&1
  echo "== col view=$v"; python tools/launch_summary.py gpurun_out/r2v_c$v.csv | head -3
done
timeout 600 python bench.py --workload sycamore --steps 3 --warmup 2 > gpurun_out/r2v_syc.jsonl 2> gpurun_out/r2v_syc.err
head -c 300 gpurun_out/r2v_syc.jsonl
